// Hardware self-test of the tcgen05 building blocks the cascade kernels rely on:
//   D[128][64] = A[off : off+128][0:64] . B[0:64][0:64]^T    (kind::tf32, fp32 accumulate)
// with both operands in the K-major SWIZZLE_NONE ("interleaved") layout
//   element (row r, k) at  (k/4)*LBO + r*16 + (k%4)*4   (SBO = 128 B, LBO = rows*16 B),
// which is linear in r, so an A operand may start at ANY row offset (the in-smem time shift).
// prep: 0 = raw fp32 bits given to the tensor core, 1 = pre-truncated to tf32, 2 = rna tf32.
#include "common.cuh"
#include "sm100.cuh"

namespace casc {
using namespace sm100;

__global__ void __launch_bounds__(128) umma_tf32_selftest_kernel(const float* A, const float* B, float* D,
                                                                 int prep, int off) {
  constexpr int RA = 144, M = 128, N = 64, K = 64;
  extern __shared__ __align__(1024) float smem_dyn[];
  float* sA = smem_dyn;
  float* sB = smem_dyn + RA * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  auto cvt = [&](float x) {
    if (prep == 1) return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    if (prep == 2) return tf32_rna(x);
    return x;
  };
  for (int e = tid; e < RA * K; e += 128) {
    int r = e / K, k = e % K;
    sA[(k / 4) * (RA * 4) + r * 4 + (k % 4)] = cvt(A[e]);
  }
  for (int e = tid; e < N * K; e += 128) {
    int n = e / K, k = e % K;
    sB[(k / 4) * (N * 4) + n * 4 + (k % 4)] = cvt(B[e]);
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<64>(&tmem_base);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = make_idesc(FMT_TF32, M, N);
    const uint32_t a0 = smem_u32(sA) + off * 16, b0 = smem_u32(sB);
#pragma unroll
    for (int ks = 0; ks < K / 8; ++ks) {    // 8 tf32 = 2 core-matrix columns per MMA
      uint64_t ad = make_sdesc(a0 + ks * 2 * (RA * 16), RA * 16, 128, LAYOUT_NONE);
      uint64_t bd = make_sdesc(b0 + ks * 2 * (N * 16), N * 16, 128, LAYOUT_NONE);
      mma_tf32(tbase, ad, bd, idesc, ks > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int row = tid;
  float v[16];
#pragma unroll
  for (int c = 0; c < N; c += 16) {
    tmem_ld16(tbase + ((uint32_t)(warp * 32) << 16) + c, v);
#pragma unroll
    for (int i = 0; i < 16; ++i) D[row * N + c + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<64>(tbase);
}

}  // namespace casc

extern "C" int casc_selftest_umma(int prep, int off, const float* A, const float* B, float* D, void* stream) {
  if (!A || !B || !D || off < 0 || off > 16 || prep < 0 || prep > 2) return CASC_ERR_ARG;
  const int smem = (144 * 64 + 64 * 64) * 4;
  cudaFuncSetAttribute(casc::umma_tf32_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  casc::umma_tf32_selftest_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(A, B, D, prep, off);
  if (cudaPeekAtLastError() != cudaSuccess) {
    (void)cudaGetLastError();
    return CASC_ERR_CUDA;
  }
  return CASC_OK;
}
