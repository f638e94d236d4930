// Exhaustive check (all 2^32 bit patterns with a finite result) that the integer forms used on the
// hot paths equal the hardware conversions: tf32 round-to-nearest-away and bf16 round-to-nearest-even.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
__global__ void k(unsigned long long* bad, uint32_t base) {
  const uint32_t u = base + blockIdx.x * blockDim.x + threadIdx.x;
  const float x = __uint_as_float(u);
  if (!isfinite(x)) return;
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  const uint32_t mine = (u + 0x1000u) & 0xFFFFE000u;
  if (isfinite(__uint_as_float(r)) && r != mine) atomicAdd(bad, 1ull);
  const __nv_bfloat16 h = __float2bfloat16_rn(x);
  const uint16_t hb = *reinterpret_cast<const uint16_t*>(&h);
  const uint16_t mb = (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
  if (isfinite(__bfloat162float(h)) && hb != mb) atomicAdd(bad + 1, 1ull);
}
int main() {
  unsigned long long* d; unsigned long long h[2];
  cudaMalloc(&d, 16); cudaMemset(d, 0, 16);
  for (uint64_t b = 0; b < (1ull << 32); b += (1ull << 30)) k<<<(1 << 30) / 256, 256>>>(d, (uint32_t)b);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("tf32 rna mismatches: %llu, bf16 rn mismatches: %llu (%s)\n", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
