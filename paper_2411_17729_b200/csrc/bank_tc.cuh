// Tensor-core bank path (SISO channels, fp32 mode): argument blocks and launchers.
#pragma once
#include "common.cuh"
#include <cuda_fp16.h>

namespace casc {

struct BankHeadArg {
  const float* u;          // [n_ch][batch][L]
  const float* krT;        // [n_ch][2][MS][128]  hi | lo of Kr^T (k' = 127 - lag; CUDA-core head)
  const __half* kr16;      // [n_ch][16][2 * MS][8] fp16 hi | lo of the scaled weights (m = 64 head, R33)
  const float* kinv;       // [n_ch][MS]          their inverse column scales 2^(e_n - 14)
  float* V;                // [n_ch][batch][L][MS]
  const int* sys_list; int n_list;
  int64_t L; int batch; int tiles_per_cta;
  // fused output (ws head, R24-R26): channels whose parts level is Kc write their parts, not v
  OutParts op;
};
// y_l = sum_b p_b(l - o_b) + d u_l from the fused output parts (common.cuh OutParts, R24-R26)
struct BankAbTailArg {
  OutParts op;
  const float* u; float* y;                    // u, y [n_ch][batch][L]
  const float* d;
  int n_ch; int64_t L; int batch;
  const int* list; int n_list;                 // optional: only channels list[0..n_list)
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
int launch_bank_stage_rp(int m, const BankStageArg& a, cudaStream_t st);
int launch_bank_tail(int m, const BankTailArg& a, cudaStream_t st);
int launch_bank_ab_tail(const BankAbTailArg& a, cudaStream_t st);
int launch_bank_derived(const double* p64, int slots, const double* Bbar, const double* C, const double* D,
                        const int* Neff, const int* Kc, double* Kr64, float* krT, double* w64, float* w32,
                        float* c32, float* d32, float* pvec, int* tri, int fold, int n, int ms, cudaStream_t st,
                        void* kr16 = nullptr, float* kinv = nullptr);

}  // namespace casc
