// Tensor-core bank path (SISO channels, fp32 mode): argument blocks and launchers.
#pragma once
#include "common.cuh"

namespace casc {

struct BankHeadArg {
  const float* u;          // [n_ch][batch][L]
  const float* krT;        // [n_ch][2][MS][128]  hi | lo of Kr^T (k' = 127 - lag)
  float* V;                // [n_ch][batch][L][MS]
  const int* sys_list; int n_list;
  int64_t L; int batch; int tiles_per_cta;
};
struct BankStageArg {
  const float* Vs; float* Vd;   // [n_ch][batch][L][MS]
  const float* P;               // pack fp32 region: [n_ch][slots][2][MS][MS]
  int k; int slots; int64_t copy_from;    // rows [copy_from, 2^k) are copies
  const int* sys_list; int n_list;
  int64_t L; int batch; int tiles_per_cta;
};
struct BankTailArg {
  const float* Va; const float* Vb; const int* parity;   // final state buffer per channel
  const float* cvec; const float* wvec; const float* d;  // [n_ch][MS], [n_ch][MS], [n_ch]
  const int* Neff;
  const float* u; float* y;                              // [n_ch][batch][L]
  int n_ch; int64_t L; int batch;
};

bool bank_tc_supported(int m);
int launch_bank_head(int m, const BankHeadArg& a, cudaStream_t st);
int launch_bank_head_ws(int m, const BankHeadArg& a, int64_t n_seq_total, cudaStream_t st);
int launch_bank_stage_ws(int m, const BankStageArg& a, cudaStream_t st);
int launch_bank_stage_rp(int m, const BankStageArg& a, cudaStream_t st);
int launch_bank_tail(int m, const BankTailArg& a, cudaStream_t st);
int launch_kr_init(const double* Bbar, double* Kr, int n, int ms, cudaStream_t st);
int launch_kr_split(const double* Kr, const int* Kc, float* krT, int n, int ms, cudaStream_t st);

}  // namespace casc
