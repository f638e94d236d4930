// Generic shifted multi-source GEMM on the CUDA cores (fp32 FFMA, fp32 accumulate).
//
// This is the shape-generic kernel of the path: every step of PAPER.md:185-229 is an
// instance of it (see kernels.cuh). It serves shapes the tcgen05 kernels do not cover
// (any m, p, q) and is the stepping stone the tensor-core kernels are checked against.
// Layout: a 64 (time rows) x 64 (outputs) tile per 256-thread block, 4x4 micro-tiles,
// K chunks of 16 staged in shared memory; rows run over batch*L of one system
// (grid.y = system list entry), the time shift stays inside each sequence.
#include "common.cuh"
#include "kernels.cuh"

namespace casc {

template <typename T>
__device__ __forceinline__ float ld_as_f32(const void* base, int64_t idx) {
  return to_f32(reinterpret_cast<const T*>(base)[idx]);
}

__global__ void __launch_bounds__(256) simt_gemm_kernel(GemmArg g) {
  const int s = g.sys_list[blockIdx.y];
  const int64_t rows = (int64_t)g.batch * g.L;
  const int64_t row0 = (int64_t)blockIdx.x * 64;
  const int col0 = blockIdx.z * 64;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;

  __shared__ float As[16][64 + 4];
  __shared__ float Ws[16][64 + 4];
  float acc[4][4] = {};

  for (int si = 0; si < g.n_src; ++si) {
    const SrcArg& sa = g.src[si];
    const int64_t shift = sa.shift_from_N ? ((int64_t)1 << g.Neff[s]) : sa.shift;
    const char* Abase = reinterpret_cast<const char*>(sa.A) +
                        (int64_t)s * sa.A_sys * (sa.a_bf16 ? 2 : 4);
    const int64_t W_off = (int64_t)s * sa.W_sys;
    const float* Wlo = sa.Wlo ? sa.Wlo + W_off : nullptr;
    for (int k0 = 0; k0 < sa.K; k0 += 16) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = tid + i * 256;
        {  // A chunk: 64 rows x 16 k
          const int r = e / 16, kk = e % 16;
          const int64_t gr = row0 + r;
          const int gk = k0 + kk;
          float v = 0.f;
          if (gr < rows && gk < sa.K) {
            const int64_t b = gr / g.L, l = gr - b * g.L, ls = l - shift;
            if (ls >= 0) {
              const int64_t idx = (b * g.L + ls) * sa.K + gk;
              v = sa.a_bf16 ? ld_as_f32<__nv_bfloat16>(Abase, idx) : ld_as_f32<float>(Abase, idx);
            }
          }
          As[kk][r] = v;
        }
        {  // W chunk: 64 outputs x 16 k, stored k-major
          const int n = e / 16, kk = e % 16;
          const int gn = col0 + n, gk = k0 + kk;
          float w = 0.f;
          if (gn < g.n_out && gk < sa.K) {
            const int64_t widx = W_off + (int64_t)gn * sa.K + gk;
            w = sa.w_bf16 ? ld_as_f32<__nv_bfloat16>(sa.W, widx) : ld_as_f32<float>(sa.W, widx);
            if (Wlo) w += Wlo[(int64_t)gn * sa.K + gk];
          }
          Ws[kk][n] = w;
        }
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        float av[4], wv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) wv[j] = Ws[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], wv[j], acc[i][j]);
      }
      __syncthreads();
    }
  }

  const int64_t R_off = (int64_t)s * g.R_sys, O_off = (int64_t)s * g.out_sys;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gr = row0 + ty * 4 + i;
    if (gr >= rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = col0 + tx * 4 + j;
      if (gn >= g.n_out) continue;
      const int64_t idx = gr * g.n_out + gn;
      float v = acc[i][j];
      if (g.R) {
        v += g.out_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(g.R)[R_off + idx])
                        : reinterpret_cast<const float*>(g.R)[R_off + idx];
      }
      if (g.out_bf16)
        reinterpret_cast<__nv_bfloat16*>(g.out)[O_off + idx] = __float2bfloat16_rn(v);
      else
        reinterpret_cast<float*>(g.out)[O_off + idx] = v;
    }
  }
}

int launch_simt_gemm(const GemmArg& g, cudaStream_t st) {
  if (g.n_list <= 0) return CASC_OK;
  const int64_t rows = (int64_t)g.batch * g.L;
  const int64_t gx = ceil_div(rows, 64);
  if (gx > 0x7fffffff || g.n_list > 65535) return CASC_ERR_UNSUPPORTED;
  dim3 grid((unsigned)gx, (unsigned)g.n_list, (unsigned)ceil_div(g.n_out, 64));
  simt_gemm_kernel<<<grid, 256, 0, st>>>(g);
  CASC_LAUNCHED();
  return CASC_OK;
}

}  // namespace casc
