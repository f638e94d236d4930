// Internal kernel interfaces of libcascade_b200.
#pragma once
#include <algorithm>
#include "common.cuh"

namespace casc {

// ---------------------------------------------------------------- float64 batched GEMM
struct DgemmArg {
  int M, N, K;
  const double* A; int64_t lda, sA, nA; const int* selA;   // A_s = A + s*sA + selA[s]*nA
  const double* B; int64_t ldb, sB, nB; const int* selB;
  double* C; int64_t ldc, sC;
  const double* Cadd; int64_t sCadd;                        // optional C += Cadd
  const int* skip_below; int level;                         // skip s if skip_below[s] < level
};
int launch_dgemm(const DgemmArg& a, int n_sys, cudaStream_t st);
// Small dependent fp64 products and their operand-format images in ONE cooperative launch
// (the MIMO derived weights, mimo_engine.cu): jobs of phase 0, grid barrier, phase 1, grid
// barrier, conversions (tf32 hi/lo planes [2][n] or bf16 [n]).
struct DJob {
  const double* A; const double* B; double* C; const double* Cadd;
  int lda, ldb, ldc, M, N, K, phase;
};
struct DConv { const double* src; void* dst; int64_t n; };
struct DerivedPlan {
  DJob jobs[8]; int n_jobs;
  DConv convs[12]; int n_convs;
  int tf32;
};
int launch_derived_coop(const DerivedPlan& plan, cudaStream_t st);
int launch_pack(const PackLayout& P, int n_sys, int N_max, int m, cudaStream_t st);
int launch_powers_sumsq(const PackLayout& P, int n_sys, int N_max, int m, double* acc, cudaStream_t st);
// a1 for ONE system with m > 64: all squarings and the packing in one cooperative launch
int launch_powers_coop(const PackLayout& P, const double* Abar, int N, int m, cudaStream_t st);
int launch_powers_small(const PackLayout& P, const double* Abar, int n_sys, int N_max, int m, cudaStream_t st);
int launch_f64_to_f32(const double* src, float* dst, int64_t n, cudaStream_t st);

// ---------------------------------------------------------------- shifted multi-source GEMM
// out[s][b][l][n] = sum_src sum_j A_src[s][b][l - shift_src(s)][j] * W_src[s][n][j]
//                   (+ R[s][b][l][n])            rows with l - shift < 0 read as zero.
// One launch covers the systems sys_list[0..n_list). shift_src(s) = shift, or 2^Neff[s]
// when shift_from_N is set. This covers every step of the path:
//   first stage (a2): sources (u, 0, Bbar), (u, 1, Abar Bbar)       -> v^(1)
//   stage k   (a4) : source  (v, 2^k, P_k), residual v                -> v^(k+1)
//   last stage (a5): sources (v, 0, C), (v, 2^N, C P_N), (u, 0, D)   -> y
struct SrcArg {
  const void* A; int64_t A_sys; int K; int a_bf16;
  const void* W; int64_t W_sys; int w_bf16;
  const float* Wlo;            // optional tf32 lo part of an fp32 W, same layout as W
  int64_t shift; int shift_from_N;
};
struct GemmArg {
  SrcArg src[3]; int n_src;
  const void* R; int64_t R_sys;
  void* out; int64_t out_sys; int out_bf16;
  int n_out; int64_t L; int batch;
  const int* sys_list; int n_list;
  const int* Neff;
};
int launch_simt_gemm(const GemmArg& g, cudaStream_t st);

}  // namespace casc
