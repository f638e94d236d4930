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
  // output fusion (ws head): channels with Neff == Kc end at the head; their epilogue writes
  // ab[seq][l] = (c . v_l, w . v_l) instead of v (null: always write v)
  const int* Neff; const int* Kc; const float* cvec; const float* wvec; float* ab;
  // R25: with fold, channels with Neff == Kc + 1 write (C v, C P_{Ne-1} v, C P_Ne v, C P_Ne P_{Ne-1} v)
  int fold = 0; const float* c1vec = nullptr; const float* c3vec = nullptr; float* abx = nullptr;
};
// y_l = a_l + b_{l - 2^Ne} + d u_l (R24; ab = (a, b)), or with the last stage folded (R25, channels
// with Neff - Kc odd when fold): y_l = a0_l + a1_{l-h} + a2_{l-2h} + a3_{l-3h} + d u_l, h = 2^(Ne-1),
// ab = (a0, a1), abx = (a2, a3); parts before l = 0 are zero
struct BankAbTailArg {
  const float* ab; const float* u; float* y;   // ab, abx [n_ch][batch][L][2]; u, y [n_ch][batch][L]
  const float* abx = nullptr;
  const float* d; const int* Neff; const int* Kc; int fold;
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

// Fused persistent bank kernel (bank_fused.cu): m = 64, every channel with Ne >= 7.
struct BankFusedArg {
  const float* u; float* y;               // [n_ch][batch][L]
  const float* krimg;                     // [n_ch][2][32][64][4] Krylov smem image (hi | lo)
  const float* cvec; const float* wvec;   // [n_ch][64]: C and w = C P_Ne (fp32)
  const float* dvec;                      // [n_ch]
  const int* order; const int* Neff;      // processing order (Ne descending), effective orders
  unsigned* flags;                        // [S][ntiles] publication flags (zeroed per launch)
  unsigned* done;                         // [n_list*batch] completed chunks per sequence (zeroed)
  const float* pub;                       // [S][NL][ntiles*128][64] publication planes
  int64_t L; int batch; int ntiles; int T; int nchunk; int S; int NL; int planes_per_ch;
  int64_t total_chunks; int discard;
  unsigned long long* dbg;                // optional [24] wait-cycle counters (CASC_FUSED_DBG=1)
};
int launch_kr_image(const double* Kr, const int* Kc, float* img, int n, cudaStream_t st);
int launch_bank_fused(const BankFusedArg& a, const float* pack_f32, int n_planes_total, int grid, cudaStream_t st);

bool bank_tc_supported(int m);
int launch_bank_head(int m, const BankHeadArg& a, cudaStream_t st);
int launch_bank_head_ws(int m, const BankHeadArg& a, int64_t n_seq_total, cudaStream_t st);
int launch_bank_stage_ws(int m, const BankStageArg& a, cudaStream_t st);
int launch_bank_stage_rp(int m, const BankStageArg& a, cudaStream_t st);
int launch_bank_tail(int m, const BankTailArg& a, cudaStream_t st);
int launch_bank_ab_tail(const BankAbTailArg& a, cudaStream_t st);
int launch_kr_init(const double* Bbar, double* Kr, int n, int ms, cudaStream_t st);
int launch_bank_derived(const double* p64, int slots, const double* Bbar, const double* C, const double* D,
                        const int* Neff, const int* Kc, double* Kr64, float* krT, double* w64, float* w32,
                        float* c32, float* d32, float* c1_32, float* c3_32, int n, int ms, cudaStream_t st);
int launch_kr_split(const double* Kr, const int* Kc, float* krT, int n, int ms, cudaStream_t st);

}  // namespace casc
