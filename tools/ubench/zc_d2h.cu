// Microbenchmark (diagnostics, not part of the library): device -> pinned host copy of a scattered
// list of channels (262 KB each) by (a) one cudaMemcpyAsync per channel, (b) one kernel storing
// straight into the mapped pinned buffer (zero-copy over PCIe), for several grid sizes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench/zc_d2h.cu -o zc_d2h
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>

__global__ void zc_copy(const float4* __restrict__ src, float4* dst, const int* list, int n_list, int64_t row4) {
  const int64_t total = (int64_t)n_list * row4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = list[i / row4];
    const int64_t o = (int64_t)c * row4 + i % row4;
    dst[o] = src[o];
  }
}
__global__ void spin(long long cycles) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
}

int main() {
  const int n = 256, nl = 86;
  const int64_t row = 4 * 16384;              // floats per channel (batch 4 x L 16384)
  float *d, *h;
  cudaMalloc(&d, n * row * 4);
  cudaHostAlloc(&h, n * row * 4, cudaHostAllocDefault);
  cudaMemset(d, 0, n * row * 4);
  std::vector<int> perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  std::shuffle(perm.begin(), perm.end(), std::mt19937(0));
  perm.resize(nl);
  int* dl;
  cudaMalloc(&dl, nl * 4);
  cudaMemcpy(dl, perm.data(), nl * 4, cudaMemcpyHostToDevice);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](auto fn) {
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      spin<<<1, 1, 0, s>>>(20000000);
      cudaEventRecord(a, s); fn(); cudaEventRecord(b, s); cudaEventSynchronize(b);
      float t; cudaEventElapsedTime(&t, a, b); best = std::min(best, t);
    }
    return best;
  };
  printf("memcpy per channel: %.3f ms\n", timeit([&] {
    for (int c : perm) cudaMemcpyAsync(h + c * row, d + c * row, row * 4, cudaMemcpyDeviceToHost, s);
  }));
  printf("one memcpy (same bytes): %.3f ms\n", timeit([&] { cudaMemcpyAsync(h, d, nl * row * 4, cudaMemcpyDeviceToHost, s); }));
  for (int g : {8, 16, 32, 64, 148, 296}) {
    printf("zero-copy kernel grid %3d: %.3f ms (%s)\n", g, timeit([&] {
      zc_copy<<<g, 512, 0, s>>>((const float4*)d, (float4*)h, dl, nl, row / 4);
    }), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
