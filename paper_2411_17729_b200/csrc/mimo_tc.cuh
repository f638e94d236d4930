// Tensor-core shifted multi-source GEMM (MIMO steps and bank streaming stages): argument
// blocks and launchers (internal).
#pragma once
#include <cuda.h>
#include "common.cuh"

namespace casc {

constexpr int kMaxSrc = 5;        // sources of one shifted GEMM (MIMO head: four lags; folded output: 4 + D)
struct MimoMaps {                 // passed as one __grid_constant__ kernel parameter
  CUtensorMap A[kMaxSrc];         // source signals [seq][L][K_src]    box {128 B, 128, 1}
  CUtensorMap W[kMaxSrc];         // weight planes [plane][n_out][K]   box {128 B, BN, 1}
  CUtensorMap R;                  // residual [seq][L][n_out]          box {128 B, 128, 1}
  CUtensorMap out;                // output   [seq][L][n_out]          box {128 B, 128, 1}
};
struct MimoArg {
  int n_src; int K[kMaxSrc]; int64_t shift[kMaxSrc]; int w_plane_off[kMaxSrc]; int w_plane_stride[kMaxSrc];
  int64_t L; int batch; int n_out; int has_residual;
  const int* sys_list; int n_list;   // systems processed (bank channels); null: one system
  int t_first;                       // first 128-step time tile processed in each sequence
  int a_row0[kMaxSrc], r_row0, out_row0;   // rows in front of local row 0 (sequence-shard halo)
  // Bank output fusion (fp32 n_out = 64): for systems with ab_neff[sys] == ab_level this stage
  // is their last streaming stage; instead of storing v^(Ne) the epilogue writes
  // ab planes (c . v_l, w . v_l) with c = C, w = C P_Ne (R24)
  const int* ab_neff; int ab_level; const float* ab_c; const float* ab_w; float* ab; int64_t ab_plane;
  int64_t gt;                        // tiles per block of the CTA tile walk
  unsigned long long* dbg;           // optional wait-cycle counters (CASC_GEMM_DBG=1)
  int64_t perm_j;                    // time-tile order within a sequence (0: natural), see decode()
  // sequence-sharded peer halo (CASC_HALO_PEER, seqshard.cu): output rows l >= peer_l_begin are also
  // stored into the successor rank's buffer of the same layout, at storage row out_row0 + l -
  // peer_shift (its halo rows), through a peer-mapped pointer (CTA-pair kernels only)
  void* peer_out; int64_t peer_l_begin, peer_shift;
};
struct MimoSrc {
  const void* A; const void* W; int K; int64_t shift;
  int w_plane_off = 0;               // plane of this source's (hi) weight for system 0
  int w_plane_stride = 0;            // weight planes per system (bank: slots * 2; 0: shared)
  int64_t w_planes = 0;              // planes in W (0: 1 for bf16, 2 for 3xTF32)
  int64_t row0 = 0;                  // halo rows stored in front of local row 0 of A
};
struct MimoGemm {
  MimoSrc src[kMaxSrc]; int n_src;
  const void* R; void* out; int n_out;
  int64_t L; int batch;
  const int* sys_list = nullptr; int n_list = 1; int n_sys_total = 1;
  int t_first = 0;
  int64_t R_row0 = 0, out_row0 = 0;  // halo rows in front of local row 0 of R / out
  int w_resident = 0;                // keep the weights in shared memory across tiles
  const int* ab_neff = nullptr; int ab_level = -1;    // see MimoArg
  const float* ab_c = nullptr; const float* ab_w = nullptr; float* ab = nullptr;
  int64_t ab_plane = 0;              // ab holds two planes: (c . v) at ab[r], (w . v) at ab[ab_plane + r]
  // general fused output (R24-R26, common.cuh) for the history-resident stage kernel; parts_deep:
  // some channel of this pass writes more than the two R24 parts (the multi-source GEMM cannot)
  OutParts parts; int parts_deep = 0;
  // bank stage kernel only (bank_hist.cu): per-system lower-triangular weight flags (the zero upper
  // blocks are skipped, NEXT-3) and the profiler's issued-flop counter
  const int* tri = nullptr;
  unsigned long long* flop_counter = nullptr;
  // see MimoArg::peer_out (the CTA-pair kernels; other kernels report CASC_ERR_UNSUPPORTED)
  void* peer_out = nullptr; int64_t peer_l_begin = 0, peer_shift = 0;
};

// Tile order of the CTA-pair GEMMs (mimo_tc2.cu, mimo_tc3.cu): pair p walks t = p, p + P, ... and
// t maps to the physical tile T = row block * n_nblk + column block. In full groups of P * n_nblk
// tiles, pair p takes the n_nblk column blocks of ONE row block back to back (T = g*P*n_nblk +
// p*n_nblk + nb), so the row block's A operand is re-read by the same SM pair while it is in its
// die's L2 instead of by n_nblk pairs spread over both dies; the last partial group keeps the
// identity order. A bijection of [0, n_tiles) either way.
__device__ __forceinline__ int64_t pair_tile_order(int64_t t, int64_t n_pairs, int n_nblk, int64_t n_tiles) {
#ifdef CASC_PAIR_NATURAL_ORDER
  return t;
#else
  const int64_t G = n_pairs * n_nblk, g = t / G;
  if ((g + 1) * G > n_tiles) return t;
  const int64_t u = t - g * G;
  return g * G + (u % n_pairs) * n_nblk + u / n_pairs;
#endif
}

bool mimo_tc_supported(int m, int p, int q);
// 3-D tensor map [d2][d1][d0] (d0 contiguous), box {128 B, rows, 1}, SWIZZLE_128B (fp32 or bf16)
bool map3d(CUtensorMap* m, const void* base, bool f32, int64_t d0, int64_t d1, int64_t d2, int rows);
// tf32 = true: 3xTF32 (fp32 signals, weights as tf32 hi/lo planes); else bf16.
int launch_mimo_gemm(const MimoGemm& g, bool tf32, cudaStream_t st);
// Bank stage pass with the state history resident in shared memory (bank_hist.cu): m = 64 fp32,
// 1 or 3 sources v at shifts c * s (s a multiple of 128); CASC_ERR_UNSUPPORTED otherwise.
int launch_bank_hist(const MimoGemm& g, cudaStream_t st);
// whether launch_bank_hist takes a pass with these parameters (the engine plans R25 with it)
bool bank_hist_ok(int64_t L, int64_t shift, int n_src, int t_first);
// bf16, n_out % 256 == 0, one system: 256 x 256 tiles on CTA pairs (mimo_tc2.cu)
bool mimo_pair_ok(const MimoGemm& g, bool tf32);
int launch_mimo_gemm_pair(const MimoGemm& g, cudaStream_t st);
// 3xTF32, n_out % 64 == 0, one system: 256 x 64|128 tiles on CTA pairs (mimo_tc3.cu)
bool mimo_pair_tf32_ok(const MimoGemm& g);
int launch_mimo_gemm_pair_tf32(const MimoGemm& g, cudaStream_t st);

}  // namespace casc
