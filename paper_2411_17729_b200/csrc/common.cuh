// Shared device/host helpers of libcascade_b200 (internal; not part of the C ABI).
#pragma once
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/cascade.h"

namespace casc {

// per-host-thread launch counter (casc_last_launch_count)
extern thread_local int g_launches;
inline void count_launch(int n = 1) { g_launches += n; }

#define CASC_TRY(expr)                                      \
  do {                                                      \
    cudaError_t e__ = (expr);                               \
    if (e__ != cudaSuccess) return CASC_ERR_CUDA;           \
  } while (0)

// diagnostics (CASC_SYNC_DEBUG=1): synchronise after every launch and name the failing one
inline bool sync_debug() {
  static const bool on = getenv("CASC_SYNC_DEBUG") != nullptr;
  return on;
}
inline void sync_check(const char* file, int line) {
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) fprintf(stderr, "casc: launch at %s:%d failed: %s\n", file, line, cudaGetErrorString(e));
}
#define CASC_LAUNCHED()                                     \
  do {                                                      \
    ::casc::count_launch();                                 \
    if (::casc::sync_debug()) ::casc::sync_check(__FILE__, __LINE__); \
    if (cudaPeekAtLastError() != cudaSuccess) {             \
      (void)cudaGetLastError();                             \
      return CASC_ERR_CUDA;                                 \
    }                                                       \
  } while (0)

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
// Effective order for length L (R20): stages with 2^k >= L are identities, so
// Ne = min(N, floor(log2(L - 1))) (0 for L <= 2) -- the last stage actually applied.
inline int eff_order(int N, int64_t L) {
  if (L <= 2) return 0;
  int kstar = 0;                                   // largest k with 2^k < L
  while (((int64_t)1 << (kstar + 1)) < L) ++kstar;
  return N < kstar ? N : kstar;
}
// Fused output of a bank channel's last stages (R24-R26). y is linear in the state, so
// the kernel producing v' = v^(Ne-d) writes the 2^(d+1) row scalars p_b = (C prod_{i in b} P_{j_i}) . v'
// over the subsets b of the stages j_i = Ne-d+i (i = 0..d; stage Ne is the tail's, R21), and the
// tail forms y_l = sum_b p_b(l - o_b) + D u_l with o_b = sum_{i in b} 2^{j_i}.
//   d = 0 (R24): the pass producing v^(Ne); d = 1 (R25): Ne - Kc odd, the single-stage pass is
//   skipped; d = 2 (R26): Ne - Kc even >= 2, the channel's last stage-pair pass is skipped.
constexpr int kMaxParts = 8;
__host__ __device__ inline int fold_depth(int ne, int kc, int fold) {   // fold: 0 (R24) | 1 (R25) | 2 (R26)
  return (!fold || ne == kc) ? 0 : (((ne - kc) & 1) ? 1 : (fold >= 2 ? 2 : 0));
}
struct OutParts {
  float* planes = nullptr;          // [kMaxParts][plane]: part b of row r at planes[b * plane + r]
  int64_t plane = 0;                // rows per plane (channels x batch x L)
  const float* vec = nullptr;       // [n_ch][kMaxParts][64] fp32 row vectors
  const int* neff = nullptr;        // per channel Ne and head stages Kc (device)
  const int* kc = nullptr;
  int fold = 0;                     // d = fold_depth(Ne, Kc, fold)
  int level = -1;                   // state level this launch produces: channels with Ne - d == level write
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bump allocator used both to size (base == nullptr) and to carve a workspace.
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base(static_cast<char*>(b)) {}
  template <class T>
  T* take(size_t count) {
    off = align_up(off, 256);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
  size_t bytes() const { return align_up(off, 256); }
};

// Pack layout (opaque to callers):
//   header  : int N_s[n_sys]
//   p64     : double [n_sys][N_max+1][m][m]          float64 powers P_k = Abar^(2^k)
//   fp32    : float  [n_sys][N_max+1][2][m][m]       tf32 hi, tf32 lo   (mode FP32)
//   bf16    : bf16   [n_sys][N_max+1][m][m]          (mode BF16)
struct PackLayout {
  int* hdr;
  double* p64;
  float* f32;
  __nv_bfloat16* b16;
  size_t bytes;
};

inline PackLayout pack_layout(void* pack, int n_sys, int m, int N_max, int mode) {
  Carver c(pack);
  PackLayout L{};
  const size_t mm = (size_t)m * m, slots = (size_t)n_sys * (N_max + 1);
  L.hdr = c.take<int>(n_sys);
  L.p64 = c.take<double>(slots * mm);
  L.f32 = nullptr;
  L.b16 = nullptr;
  // tf32 hi/lo planes in fp32 mode, and also in bf16 mode for m <= 64 (bank sizes: the bf16 SISO
  // bank runs the fp32 tensor-core bank path, cascade_api.cu); the fp32-mode layout is a prefix
  if (mode == CASC_FP32 || m <= 64) L.f32 = c.take<float>(slots * 2 * mm);
  if (mode != CASC_FP32) L.b16 = c.take<__nv_bfloat16>(slots * mm);
  L.bytes = c.bytes();
  return L;
}

__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }

// Round to tf32 (10 explicit mantissa bits), nearest with ties away from zero: add half a tf32
// ulp to the magnitude bits and clear the 13 dropped bits. Bitwise equal to cvt.rna.tf32.f32
// for every finite input (checked exhaustively on B200, tools/ubench/cvt_check.cu) but on the
// integer pipe: cvt runs on the XU pipe, which bounded the split warps of the 3xTF32 kernels.
__device__ __forceinline__ float tf32_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
// 3xTF32 split of a streaming fp32 operand (R17): hi = rna_tf32(x), lo = rna_tf32(x - hi)
// (x - hi is exact in fp32), so x = hi + lo to ~2^-23 relative with an unbiased rounding.
__device__ __forceinline__ float4 tf32_hi4(float4 v) {
  return make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
}
// The tf32 part the tensor core reads from an fp32 operand in shared memory: the top 19 bits
// (truncation; checked on B200: a remainder computed against round-to-nearest would be off by an
// ulp and fails the 1e-5 parity). With A_hi left as the raw fp32 chunk, lo = rna(v - trunc(v)).
__device__ __forceinline__ float4 tf32_trunc4(float4 v) {
  return make_float4(__uint_as_float(__float_as_uint(v.x) & 0xffffe000u), __uint_as_float(__float_as_uint(v.y) & 0xffffe000u),
                     __uint_as_float(__float_as_uint(v.z) & 0xffffe000u), __uint_as_float(__float_as_uint(v.w) & 0xffffe000u));
}
__device__ __forceinline__ float4 tf32_lo4(float4 v, float4 h) {
  return make_float4(tf32_rna(v.x - h.x), tf32_rna(v.y - h.y), tf32_rna(v.z - h.z), tf32_rna(v.w - h.w));
}

}  // namespace casc
