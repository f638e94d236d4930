// Shifted multi-source GEMM on the sm_100a tensor cores: every dense cascade step.
//
// One kernel computes the steps of PAPER.md:185-229 as
//   out[s][l][n] = sum_src sum_k A_src[s][l - shift_src][k] W_src(s)[n][k]  (+ R[s][l][n])
// over sequences s (a (system, batch) pair) and time steps l:
//   MIMO first stage (a2): (u, 0, Bbar), (u, 1, Abar Bbar)            -> v^(1)
//   MIMO / bank stage (a4): (v, 2^k, Abar^(2^k)) + residual v          -> v^(k+1)
//   MIMO last stage  (a5): (v, 0, C), (v, 2^N, C Abar^(2^N)), (u, 0, D) -> y
// The time shift is a TMA coordinate offset; rows l - shift < 0 fall outside the tensor and
// TMA zero-fills them, which is exactly "columns l < 2^k are left unchanged".
// For a bank of channels the weight W_src(s) is the power of the channel owning sequence s:
// the weight tensor is a stack of planes and each tile selects its plane.
//
// Two precisions (template TF32):
//   bf16   : kind::f16, bf16 tiles of 128 x 64 (128-B rows), fp32 accumulation, bf16 output.
//   3xTF32 : kind::tf32 with hi.hi + lo.hi + hi.lo, fp32 tiles of 128 x 32 (128-B rows). W comes
//            as tf32 hi/lo planes; transform warps split the landed A tile in shared memory into
//            hi = rna(x) (in place) and lo = rna(x - hi). hi.hi and the two correction products
//            accumulate in separate TMEM accumulators (see ACOLS below).
//
// Persistent CTAs (one per SM):
//   warp 0      TMA producer: ring of {A, W (hi[, lo])} tiles (SWIZZLE_128B) and a separate ring
//               of residual / staging chunks (128 rows x 128 B) fetched ahead of the epilogue
//   warp 1      MMA issuer: M=128, N=BN, into one of two TMEM accumulator buffers
//   warps 2-5   epilogue: TMEM -> registers (lane = time row), + residual chunk, convert in place,
//               TMA store; accumulator released to warp 1, chunk slot released to warp 0.
//   warps 6-9   (3xTF32 only) hi/lo split of each landed A tile.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"
#include "mimo_tc.cuh"

namespace casc {
using namespace sm100;

namespace {
constexpr int BM = 128;

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];"
               ::"l"(map), "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void prefetch_map(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(m) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
        "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
        "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// fp32 pair -> bf16x2, round to nearest even (F2FP). An integer-pipe version (bitwise equal,
// tools/ubench/cvt_check.cu) was measured slower here: 2.19 vs 2.09 ms per E4 stage launch.
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_bf16(uint32_t u) {
  __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&u);
  return __bfloat1622float2(h);
}

// Compile-time configuration. WCH > 0 selects the weight-resident mode: all K chunks of the
// tile's weights (WCH at most) stay in a dedicated buffer and are reloaded only when the system
// (bank channel) changes, so the ring carries A tiles only; 3xTF32 then splits into a separate
// 2-slot lo ring. Used for the bank streaming stage, where one channel's P_k serves hundreds of
// tiles and the bytes in flight decide the DRAM throughput.
template <int BN, bool TF32, int RSO = 0, int WCH = 0>
struct Cfg {
  static constexpr bool WRES = WCH > 0;
  static constexpr int ES = TF32 ? 4 : 2;                 // element size
  static constexpr int BK = 128 / ES;                     // K per chunk: 128-byte rows
  static constexpr uint32_t A_BYTES = BM * 128;           // 16 KB
  static constexpr uint32_t W_BYTES = BN * 128;           // one of hi / lo
  static constexpr int NW = TF32 ? 2 : 1;                 // weight tiles per chunk
  // TSA: 3xTF32 with the A operand (tf32 hi | lo) in TMEM, written by the transform warps
  // (N = 64 tiles: the two accumulator buffers leave room for two A units of 64 columns).
  // An SS tf32 MMA at N = 64 reads 6 KB of shared memory (48 cycles at 128 B/cycle vs the
  // 32-cycle floor); with A in TMEM only W is read from shared memory.
  static constexpr bool TSA = TF32 && BN == 64;
  static constexpr uint32_t STAGE_BYTES =                 // ring slot: A[, A lo][, W hi[, W lo]]
      WRES ? A_BYTES : A_BYTES * ((TF32 && !TSA) ? 2 : 1) + W_BYTES * NW;
  static constexpr uint32_t TMA_BYTES = WRES ? A_BYTES : A_BYTES + W_BYTES * NW;
  static constexpr uint32_t WBUF = WRES ? (uint32_t)WCH * NW * W_BYTES : 0;
  static constexpr int ALO = (WRES && TF32 && !TSA) ? 2 : 0;   // separate lo slots (weight-resident SS)
  static constexpr int RS = RSO ? RSO : ((TF32 && BN == 64) ? 4 : 2);   // residual / staging chunks
  static constexpr uint32_t R_BYTES = BM * 128;           // 16 KB
  static constexpr int STAGES_FIT =
      (int)((226u * 1024u - 1024u - RS * R_BYTES - WBUF - ALO * A_BYTES) / STAGE_BYTES);
  static constexpr int STAGES = STAGES_FIT < 8 ? STAGES_FIT : 8;
  static constexpr int CW = 128 / ES;                     // epilogue chunk width (columns)
  static constexpr int R_WARP = TF32 ? 10 : 6;            // residual / staging producer warp
  static constexpr int THREADS = 32 * (R_WARP + 1);
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + WBUF + ALO * A_BYTES + RS * R_BYTES;
};

// Tile -> (sequence coordinate in the tensors, time tile, N block, system)
struct TileCoord {
  int seq, l0, nb, sys;
};
__device__ __forceinline__ TileCoord decode(int64_t tile, const MimoArg& a, int n_nblk, int64_t nt_eff) {
  TileCoord t;
  t.nb = (int)(tile % n_nblk);
  const int64_t r = tile / n_nblk;
  // Time tiles in residue-class order: with S = nt_eff / perm_j (the smallest shift in tiles),
  // position q holds tile (q % perm_j) * S + q / perm_j, so the tiles reading a row (as the
  // residual and at shifts S, 2S, 3S) follow each other and the row is fetched from DRAM once.
  int64_t q = r % nt_eff;
  if (a.perm_j) q = (q % a.perm_j) * (nt_eff / a.perm_j) + q / a.perm_j;
  t.l0 = (int)((a.t_first + q) * BM);
  const int64_t sidx = r / nt_eff;
  const int li = (int)(sidx / a.batch), b = (int)(sidx % a.batch);
  const int sys = a.sys_list ? a.sys_list[li] : 0;
  t.seq = sys * a.batch + b;
  t.sys = sys;
  return t;
}

// The CTA's walk over tiles: blocks of gt consecutive tiles dealt round-robin over the grid
// (gt = 1: plain round-robin; weight-resident mode: one contiguous range per CTA, so a CTA
// reloads its resident weights only where its range crosses a system boundary). Every role
// runs its own copy of the same walk.
struct Walk {
  int64_t blk, i, n_tiles, gt;
  __device__ Walk(int64_t n, int64_t g) : blk(blockIdx.x), i(0), n_tiles(n), gt(g) {}
  __device__ bool valid() const { return blk * gt + i < n_tiles; }
  __device__ int64_t tile() const { return blk * gt + i; }
  __device__ void next() {
    if (++i == gt || blk * gt + i >= n_tiles) { i = 0; blk += gridDim.x; }
  }
};
}  // namespace

template <int BN, bool TF32, int RSO = 0, int WCH = 0>
__global__ void __launch_bounds__(Cfg<BN, TF32, RSO, WCH>::THREADS, 1)
    mimo_gemm_kernel(const __grid_constant__ MimoMaps maps, MimoArg a) {
  using C = Cfg<BN, TF32, RSO, WCH>;
  constexpr bool WRES = C::WRES;
  constexpr int STAGES = C::STAGES, BK = C::BK, RS = C::RS;
  static_assert(STAGES >= 2, "shared memory too small for a 2-deep ring");
  // TMEM: two accumulator buffers of ACOLS columns. 3xTF32 keeps hi.hi in [0, BN) ("main") and
  // the two correction products in [BN, 2BN) ("corr"): the tensor core's fp32 accumulator
  // truncates at every MMA, so the error grows with the number of MMAs chained into one
  // accumulator (measured ~2e-8 per MMA); splitting keeps the main chain at K/8 MMAs and the
  // corr chain's error is 2^-11 smaller. The epilogue sums main + corr with round-to-nearest.
  constexpr int ACOLS = TF32 ? 2 * BN : BN;
  constexpr bool TSA = C::TSA;
  constexpr uint32_t AU0 = 2 * ACOLS;                        // TSA: first A unit (hi | lo, 64 columns)
  // A units (TSA: TMEM, 64 columns each; weight-resident SS: shared-memory lo slots): with four
  // units the transform of chunk j + 2 no longer waits for the MMAs of chunk j to complete
  constexpr int NAU_SH = TSA ? 2 : 1, NAU = 1 << NAU_SH;
  constexpr int TUSED = 2 * ACOLS + (TSA ? 64 * NAU : 0);
  static_assert(TUSED <= 512, "TMEM holds 512 columns");
  constexpr int TCOLS = TUSED <= 32 ? 32 : TUSED <= 64 ? 64 : TUSED <= 128 ? 128 : TUSED <= 256 ? 256 : 512;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps the shared state space (STS/LDS, not generic ST/LD)
  uint8_t* sWres = smem + STAGES * C::STAGE_BYTES;           // [WCH][hi, lo] (weight-resident)
  uint8_t* sAlo = sWres + C::WBUF;                           // [ALO] (weight-resident 3xTF32)
  uint8_t* sR = sAlo + C::ALO * C::A_BYTES;                  // [RS][R_BYTES]
  constexpr int NLO = (WRES || TSA) ? NAU : STAGES;            // lo_ready barriers
  __shared__ uint64_t full[STAGES], empty[STAGES], lo_ready[NLO], alo_free[NAU], tfull[2], tempty[2],
      rfull[RS], rempty[RS], w_full, wfree;
  __shared__ uint32_t tmem_base;
  auto stA = [&](int s) { return smem + s * C::STAGE_BYTES; };
  auto stW = [&](int s) { return smem + s * C::STAGE_BYTES + C::A_BYTES; };
  auto stWlo = [&](int s) { return smem + s * C::STAGE_BYTES + C::A_BYTES + C::W_BYTES; };
  auto stAlo = [&](int s) { return smem + s * C::STAGE_BYTES + C::A_BYTES + C::NW * C::W_BYTES; };

  // warp index broadcast from lane 0: provably warp-uniform, so role branches are uniform control
  // flow and ptxas keeps role-local uniform values (descriptors, TMEM addresses) in uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  // optional wait-cycle accounting (a.dbg != null, CASC_GEMM_DBG=1): slots per role, see launcher
  unsigned long long dacc[24];
#pragma unroll
  for (int i = 0; i < 24; ++i) dacc[i] = 0;
  const long long t_start = clock64();
#define TWM(slot, stmt)                                      \
  do {                                                       \
    if (a.dbg) {                                             \
      const long long t0_ = clock64();                       \
      stmt;                                                  \
      dacc[slot] += (unsigned long long)(clock64() - t0_);   \
    } else {                                                 \
      stmt;                                                  \
    }                                                        \
  } while (0)
  const int64_t mt_per_b = (a.L + BM - 1) / BM;
  const int64_t nt_eff = mt_per_b - a.t_first;
  const int n_nblk = (a.n_out + BN - 1) / BN;
  const int64_t n_tiles = (int64_t)a.n_list * a.batch * nt_eff * n_nblk;
  constexpr int NCH = BN / C::CW;                   // epilogue chunks per tile

  if (threadIdx.x == 0) {
    // TSA + resident weights: a ring slot (A only) is free once the transform warps have read it
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], (TSA && WRES) ? 128 : 1); }
    for (int s = 0; s < NLO; ++s) mbar_init(&lo_ready[s], 128);
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 128); }
    for (int s = 0; s < NAU; ++s) mbar_init(&alo_free[s], 1);
    for (int s = 0; s < RS; ++s) { mbar_init(&rfull[s], 1); mbar_init(&rempty[s], 1); }
    mbar_init(&w_full, 1);
    mbar_init(&wfree, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<TCOLS>(&tmem_base);
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < a.n_src; ++s) { prefetch_map(&maps.A[s]); prefetch_map(&maps.W[s]); }
    prefetch_map(&maps.out);
    if (a.has_residual) prefetch_map(&maps.R);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // A CTA that allocates all 512 columns owns the whole TMEM, so its base is column 0, lane 0.
  // Using the constant keeps every TMEM operand address a compile-time value: loaded from shared
  // memory it lives in per-thread registers and each MMA issue pays R2UR conversions.
  if (TCOLS == 512 && tmem_base != 0) __trap();
  const uint32_t tbase = TCOLS == 512 ? 0u : tmem_base;

  // Producer loops run on the whole warp and only lane 0 issues: a loop inside a lane-divergent
  // region makes ptxas keep every role's loop-carried values in per-thread registers, and the MMA
  // warp then pays R2UR conversions for each MMA operand (measured: 49 per 12-MMA chunk, 0 this way).
  if (warp == 0) {
    // =========================================================== TMA producer
    {
      const bool issue = lane == 0;
      int s = 0, cur_sys = -1, n_reload = 0;
      uint32_t ph = 0;
      for (Walk w(n_tiles, a.gt); w.valid(); w.next()) {
        const TileCoord tc = decode(w.tile(), a, n_nblk, nt_eff);
        if (WRES && tc.sys != cur_sys) {
          // every MMA with the previous weights must be complete (the MMA warp commits wfree when it
          // meets the system change)
          if (n_reload > 0) TWM(0, mbar_wait(&wfree, (uint32_t)((n_reload - 1) & 1)));
          ++n_reload;
          uint32_t bytes = 0;
          for (int src = 0; src < a.n_src; ++src) bytes += (uint32_t)(a.K[src] / BK) * C::NW * C::W_BYTES;
          if (issue) mbar_arrive_expect_tx(&w_full, bytes);
          int ci = 0;
          for (int src = 0; src < a.n_src; ++src) {
            const int plane = tc.sys * a.w_plane_stride[src] + a.w_plane_off[src];
            for (int kc = 0; kc < a.K[src] / BK; ++kc, ++ci) {
              uint8_t* wdst = sWres + ci * C::NW * C::W_BYTES;
              if (issue) {
                tma_load_3d(wdst, &maps.W[src], &w_full, kc * BK, tc.nb * BN, plane);
                if (TF32) tma_load_3d(wdst + C::W_BYTES, &maps.W[src], &w_full, kc * BK, tc.nb * BN, plane + 1);
              }
            }
          }
          cur_sys = tc.sys;
        }
        for (int src = 0; src < a.n_src; ++src) {
          const int nk = a.K[src] / BK;
          const int plane = tc.sys * a.w_plane_stride[src] + a.w_plane_off[src];
          for (int kc = 0; kc < nk; ++kc) {
            TWM(1, mbar_wait(&empty[s], ph ^ 1));
            if (issue) {
              mbar_arrive_expect_tx(&full[s], C::TMA_BYTES);
              tma_load_3d(stA(s), &maps.A[src], &full[s], kc * BK, a.a_row0[src] + tc.l0 - (int)a.shift[src], tc.seq);
              if (!WRES) {
                tma_load_3d(stW(s), &maps.W[src], &full[s], kc * BK, tc.nb * BN, plane);
                if (TF32) tma_load_3d(stWlo(s), &maps.W[src], &full[s], kc * BK, tc.nb * BN, plane + 1);
              }
            }
            if (++s == STAGES) { s = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == C::R_WARP) {
    // =========================================================== residual / staging producer
    {
      const bool issue = lane == 0;
      int rs = 0;
      uint32_t rph = 0;
      for (Walk w(n_tiles, a.gt); w.valid(); w.next()) {
        const TileCoord tc = decode(w.tile(), a, n_nblk, nt_eff);
        for (int j = 0; j < NCH; ++j) {
          TWM(20, mbar_wait(&rempty[rs], rph ^ 1));
          if (issue) {
            if (a.has_residual) {
              mbar_arrive_expect_tx(&rfull[rs], C::R_BYTES);
              tma_load_3d(sR + rs * C::R_BYTES, &maps.R, &rfull[rs], tc.nb * BN + j * C::CW, a.r_row0 + tc.l0, tc.seq);
            } else {
              mbar_arrive(&rfull[rs]);
            }
          }
          if (++rs == RS) { rs = 0; rph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // =========================================================== MMA issuer (whole warp, elected lane issues)
    {
      const uint32_t idesc = make_idesc(TF32 ? FMT_TF32 : FMT_BF16, BM, BN);
      const uint32_t idesc128 = make_idesc(FMT_TF32, BM, 2 * BN);   // TSA: A hi x [W hi | W lo]
      int s = 0, cur_sys = -1;
      uint32_t ph = 0, wph = 0;
      int64_t t_local = 0, j = 0;                 // tiles / chunks consumed by this CTA
      int nch_tile = 0;                           // K chunks per tile, all sources in order
#pragma unroll
      for (int q = 0; q < kMaxSrc; ++q) if (q < a.n_src) nch_tile += a.K[q] / BK;
      for (Walk w(n_tiles, a.gt); w.valid(); w.next(), ++t_local) {
        // the issuing warp needs the tile's system only for resident weights (the decode costs
        // integer divisions and a list load per tile on the MMA warp's critical loop)
        const int tsys = WRES ? decode(w.tile(), a, n_nblk, nt_eff).sys : 0;
        const int acc = (int)(t_local & 1);
        TWM(4, mbar_wait_u(&tempty[acc], (uint32_t)((t_local >> 1) & 1) ^ 1));
        if (WRES && tsys != cur_sys) {
          if (cur_sys >= 0) mma_commit_w(&wfree);   // all MMAs issued so far used the old weights
          TWM(5, mbar_wait(&w_full, wph));
          wph ^= 1;
          cur_sys = tsys;
        }
        tc_fence_after();
        const uint32_t d = tbase + acc * ACOLS, dc = d + BN;
        bool first = true;
        for (int ci = 0; ci < nch_tile; ++ci, ++j) {
          {
            if (TF32) {
              if (WRES || TSA) TWM(6, mbar_wait_u(&lo_ready[j & (NAU - 1)], (uint32_t)((j >> NAU_SH) & 1)));
              else TWM(6, mbar_wait(&lo_ready[s], ph));
            } else {
              TWM(6, mbar_wait(&full[s], ph));
            }
            tc_fence_after();
            if constexpr (TSA) {                        // A from TMEM unit (j & (NAU - 1)): hi | lo
              const uint32_t ah = tbase + AU0 + (uint32_t)(j & (NAU - 1)) * 64, al = ah + 32;
              const uint64_t wd0 = make_sdesc(WRES ? smem_u32(sWres + ci * C::NW * C::W_BYTES) : smem_u32(stW(s)), 16, 1024,
                                              LAYOUT_SW128);
              // main: hi.hi; corr: lo.hi + hi.lo (four K-steps, one asm block)
              mma_3xtf32_ts_chunk8_w(d, dc, ah, al, wd0, idesc128, idesc, first ? 0u : 1u);
              first = false;
              if (!WRES) mma_commit_w(&empty[s]);         // the slot also holds W
              mma_commit_w(&alo_free[j & (NAU - 1)]);
              if (++s == STAGES) { s = 0; ph ^= 1; }
              continue;
            }
            const uint32_t a0 = smem_u32(stA(s));
            const uint32_t w0 = WRES ? smem_u32(sWres + ci * C::NW * C::W_BYTES) : smem_u32(stW(s));
            const uint32_t al0 = WRES ? smem_u32(sAlo + (j & (NAU - 1)) * C::A_BYTES) : smem_u32(stAlo(s));
            const uint64_t ad0 = make_sdesc(a0, 16, 1024, LAYOUT_SW128), wd0 = make_sdesc(w0, 16, 1024, LAYOUT_SW128);
            const uint64_t ald0 = make_sdesc(al0, 16, 1024, LAYOUT_SW128), wld0 = sdesc_add(wd0, C::W_BYTES);
#pragma unroll
            for (int k = 0; k < 4; ++k) {               // 4 x 32 B = one 128-B row per chunk
              const uint64_t ad = sdesc_add(ad0, k * 32), wd = sdesc_add(wd0, k * 32);
              if (TF32) {
                mma_tf32_w(d, ad, wd, idesc, first ? 0u : 1u);                      // main: hi.hi
                mma_tf32_w(dc, sdesc_add(ald0, k * 32), wd, idesc, first ? 0u : 1u); // corr: lo.hi + hi.lo
                mma_tf32_w(dc, ad, sdesc_add(wld0, k * 32), idesc, 1u);
              } else {
                mma_f16_w(d, ad, wd, idesc, first ? 0u : 1u);
              }
              first = false;
            }
            mma_commit_w(&empty[s]);
            if (WRES && TF32) mma_commit_w(&alo_free[j & (NAU - 1)]);
            if (++s == STAGES) { s = 0; ph ^= 1; }
          }
        }
        mma_commit_w(&tfull[acc]);
      }
    }
  } else if (warp >= 6) {
    // =========================================================== hi/lo split (3xTF32, warps 6-9)
    if (TF32) {
      const int t = threadIdx.x - 192;
      int s = 0;
      uint32_t ph = 0;
      int64_t j = 0;
      for (Walk w(n_tiles, a.gt); w.valid(); w.next()) {
        for (int src = 0; src < a.n_src; ++src) {
          const int nk = a.K[src] / BK;
          for (int kc = 0; kc < nk; ++kc, ++j) {
            TWM(8, mbar_wait(&full[s], ph));
            if constexpr (TSA) {                        // this thread's row -> tf32 hi | lo -> TMEM
              const int row = (warp & 3) * 32 + lane;
              const uint8_t* rr = stA(s) + row * 128;   // SW128: chunk c at (c ^ (row % 8)) * 16
              uint32_t hv[32], lv[32];
#pragma unroll
              for (int cc = 0; cc < 8; ++cc) {
                const float4 v = *reinterpret_cast<const float4*>(rr + ((cc ^ (row & 7)) * 16));
                const float4 h = tf32_hi4(v), l = tf32_lo4(v, h);
                hv[4 * cc] = __float_as_uint(h.x); hv[4 * cc + 1] = __float_as_uint(h.y);
                hv[4 * cc + 2] = __float_as_uint(h.z); hv[4 * cc + 3] = __float_as_uint(h.w);
                lv[4 * cc] = __float_as_uint(l.x); lv[4 * cc + 1] = __float_as_uint(l.y);
                lv[4 * cc + 2] = __float_as_uint(l.z); lv[4 * cc + 3] = __float_as_uint(l.w);
              }
              if (WRES) mbar_arrive(&empty[s]);         // slot read: the producer may refill it
              TWM(9, mbar_wait(&alo_free[j & (NAU - 1)], (uint32_t)(((j >> NAU_SH) & 1) ^ 1)));
              tc_fence_after();
              const uint32_t ta = tbase + ((uint32_t)((warp & 3) * 32) << 16) + AU0 + (uint32_t)(j & (NAU - 1)) * 64;
              tmem_st32(ta, hv);
              tmem_st32(ta + 32, lv);
              tmem_wait_st();
              tc_fence_before();
              mbar_arrive(&lo_ready[j & (NAU - 1)]);
              if (++s == STAGES) { s = 0; ph ^= 1; }
              continue;
            }
            if (WRES && j >= NAU) mbar_wait(&alo_free[j & (NAU - 1)], (uint32_t)(((j - NAU) >> NAU_SH) & 1));
            float4* hi = reinterpret_cast<float4*>(stA(s));
            float4* out = reinterpret_cast<float4*>(WRES ? sAlo + (j & (NAU - 1)) * C::A_BYTES : stAlo(s));
#pragma unroll
            for (int e = t; e < (int)(C::A_BYTES / 16); e += 128) {
              const float4 v = hi[e];                   // hi: the raw chunk (the MMA truncates it)
              out[e] = tf32_lo4(v, tf32_trunc4(v));
            }
            fence_async_smem();
            mbar_arrive(&lo_ready[WRES ? (int)(j & (NAU - 1)) : s]);
            if (++s == STAGES) { s = 0; ph ^= 1; }
          }
        }
      }
    }
  } else {
    // =========================================================== epilogue (warps 2..5)
    const int q = warp & 3;                       // TMEM lane quadrant of this warp
    const int row = q * 32 + lane;                // tile row = TMEM lane
    const bool leader = (warp == 2 && lane == 0);
    int64_t t_local = 0;
    int rs = 0, prev_rs = -1;
    uint32_t rph = 0;
    for (Walk w(n_tiles, a.gt); w.valid(); w.next(), ++t_local) {
      const TileCoord tc = decode(w.tile(), a, n_nblk, nt_eff);
      const int acc = (int)(t_local & 1);
      const bool to_ab = TF32 && a.ab != nullptr && a.ab_neff[tc.sys] == a.ab_level;
      float pa = 0.f, pb = 0.f;
      TWM(12, mbar_wait(&tfull[acc], (uint32_t)((t_local >> 1) & 1)));
      tc_fence_after();
      for (int j = 0; j < NCH; ++j) {
        uint8_t* rbuf = sR + rs * C::R_BYTES;
        uint32_t v[64];
        const uint32_t taddr = tbase + ((uint32_t)(q * 32) << 16) + acc * ACOLS + j * C::CW;
        tmem_ld32(taddr, v);
        tmem_ld32(taddr + (TF32 ? BN : 32), v + 32);     // 3xTF32: the corr accumulator
        tmem_wait_ld();
        if (TF32) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) + __uint_as_float(v[32 + e]));
        }
        TWM(13, mbar_wait(&rfull[rs], rph));
        uint8_t* rrow = rbuf + row * 128;          // SW128: 16-B chunk c at ((c ^ (row % 8)) * 16)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint4* p = reinterpret_cast<uint4*>(rrow + ((c ^ (row & 7)) * 16));
          if (TF32) {
            float f[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) f[e] = __uint_as_float(v[c * 4 + e]);
            if (a.has_residual) {
              const float4 r = *reinterpret_cast<const float4*>(p);
              f[0] += r.x; f[1] += r.y; f[2] += r.z; f[3] += r.w;
            }
            if (to_ab) {                            // y parts: c . v and w . v of this row
              const int col = tc.nb * BN + j * C::CW + c * 4;
              const float4 cc4 = __ldg(reinterpret_cast<const float4*>(a.ab_c + (int64_t)tc.sys * 64 + col));
              const float4 ww4 = __ldg(reinterpret_cast<const float4*>(a.ab_w + (int64_t)tc.sys * 64 + col));
              pa = fmaf(cc4.x, f[0], pa); pa = fmaf(cc4.y, f[1], pa); pa = fmaf(cc4.z, f[2], pa); pa = fmaf(cc4.w, f[3], pa);
              pb = fmaf(ww4.x, f[0], pb); pb = fmaf(ww4.y, f[1], pb); pb = fmaf(ww4.z, f[2], pb); pb = fmaf(ww4.w, f[3], pb);
            } else {
              *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
            }
          } else {
            float f[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(v[c * 8 + e]);
            if (a.has_residual) {
              const uint4 r = *p;
              const float2 r0 = unpack_bf16(r.x), r1 = unpack_bf16(r.y), r2 = unpack_bf16(r.z), r3 = unpack_bf16(r.w);
              f[0] += r0.x; f[1] += r0.y; f[2] += r1.x; f[3] += r1.y;
              f[4] += r2.x; f[5] += r2.y; f[6] += r3.x; f[7] += r3.y;
            }
            *p = make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
          }
        }
        if (j == NCH - 1) {                         // this tile's accumulator has been drained
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
        }
        fence_async_smem();
        named_sync(1, 128);
        if (to_ab) {                                // nothing stored: the slot is free now
          if (leader) {
            if (prev_rs >= 0) {
              bulk_wait_read<0>();
              mbar_arrive(&rempty[prev_rs]);
            }
            mbar_arrive(&rempty[rs]);
          }
          prev_rs = -1;
        } else {
          if (leader) {
            tma_store_3d(&maps.out, rbuf, tc.nb * BN + j * C::CW, a.out_row0 + tc.l0, tc.seq);
            bulk_commit();
            if (prev_rs >= 0) {                     // the previous chunk's store has read its slot
              bulk_wait_read<1>();
              mbar_arrive(&rempty[prev_rs]);
            }
          }
          prev_rs = rs;
        }
        if (++rs == RS) { rs = 0; rph ^= 1; }
      }
      if (to_ab) {
        const int64_t l = (int64_t)tc.l0 + row;
        if (l < a.L) {
          const int64_t r = (int64_t)tc.seq * a.L + l;
          a.ab[r] = pa;
          a.ab[a.ab_plane + r] = pb;
        }
      }
    }
    if (leader) bulk_wait<0>();
  }
  if (a.dbg) {
    if (lane == 0)
      for (int i = 0; i < 24; ++i)
        if (dacc[i]) atomicAdd(a.dbg + i, dacc[i]);
    if (threadIdx.x == 0) atomicAdd(a.dbg + 23, (unsigned long long)(clock64() - t_start));
  }
#undef TWM
  __syncthreads();
  if (warp == 1) tmem_dealloc<TCOLS>(tbase);
}

// ----------------------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D tensor [d2][d1][d0] (d0 contiguous) with a box {128-B row, rows, 1}, SWIZZLE_128B.
bool map3d(CUtensorMap* m, const void* base, bool f32, int64_t d0, int64_t d1, int64_t d2, int rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  const int64_t es = f32 ? 4 : 2;
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t strides[2] = {(cuuint64_t)(d0 * es), (cuuint64_t)(d1 * d0 * es)};
  cuuint32_t box[3] = {(cuuint32_t)(128 / es), (cuuint32_t)rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base),
            dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool mimo_tc_supported(int m, int p, int q) { return m % 64 == 0 && p % 64 == 0 && q % 64 == 0 && m >= 64; }

template <int BN, bool TF32, int RSO = 0, int WCH = 0>
static int launch_cfg(const MimoGemm& g, cudaStream_t st) {
  using C = Cfg<BN, TF32, RSO, WCH>;
  MimoMaps maps;
  memset(&maps, 0, sizeof(maps));
  MimoArg a{};
  a.n_src = g.n_src;
  a.L = g.L;
  a.batch = g.batch;
  a.n_out = g.n_out;
  a.sys_list = g.sys_list;
  a.n_list = g.sys_list ? g.n_list : 1;
  a.t_first = g.t_first;
  a.ab_neff = g.ab_neff; a.ab_level = g.ab_level; a.ab_c = g.ab_c; a.ab_w = g.ab_w; a.ab = g.ab;
  a.ab_plane = g.ab_plane;
  if (g.parts_deep || (g.ab && (!TF32 || g.n_out != 64))) return CASC_ERR_UNSUPPORTED;
  const int64_t nseq_total = (int64_t)(g.n_sys_total > 0 ? g.n_sys_total : 1) * g.batch;
  for (int s = 0; s < g.n_src; ++s) {
    if (g.src[s].K % C::BK) return CASC_ERR_UNSUPPORTED;
    a.K[s] = g.src[s].K;
    a.shift[s] = g.src[s].shift;
    a.w_plane_off[s] = g.src[s].w_plane_off;
    a.w_plane_stride[s] = g.src[s].w_plane_stride;
    a.a_row0[s] = (int)g.src[s].row0;
    if (!map3d(&maps.A[s], g.src[s].A, TF32, g.src[s].K, g.src[s].row0 + g.L, nseq_total, BM)) return CASC_ERR_CUDA;
    // weights: planes of [n_out][K] (bf16), or hi / lo planes of tf32 for 3xTF32
    const int64_t planes = g.src[s].w_planes > 0 ? g.src[s].w_planes : (TF32 ? 2 : 1);
    if (!map3d(&maps.W[s], g.src[s].W, TF32, g.src[s].K, g.n_out, planes, BN)) return CASC_ERR_CUDA;
  }
  {
    // stride of the shifts in time tiles -> tile order (decode)
    int64_t S = 0;
    for (int s = 0; s < g.n_src; ++s)
      if (g.src[s].shift > 0 && g.src[s].shift % BM == 0) S = S ? std::min<int64_t>(S, g.src[s].shift / BM) : g.src[s].shift / BM;
    const int64_t nt_eff = (g.L + BM - 1) / BM - g.t_first;
    a.perm_j = (S > 1 && nt_eff % S == 0) ? nt_eff / S : 0;
  }
  a.has_residual = g.R != nullptr;
  a.r_row0 = (int)g.R_row0;
  a.out_row0 = (int)g.out_row0;
  if (g.R && !map3d(&maps.R, g.R, TF32, g.n_out, g.R_row0 + g.L, nseq_total, BM)) return CASC_ERR_CUDA;
  if (!map3d(&maps.out, g.out, TF32, g.n_out, g.out_row0 + g.L, nseq_total, BM)) return CASC_ERR_CUDA;
  if (cudaFuncSetAttribute(mimo_gemm_kernel<BN, TF32, RSO, WCH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)C::SMEM) != cudaSuccess)
    return CASC_ERR_CUDA;
  const int64_t tiles = (int64_t)a.n_list * g.batch * (ceil_div(g.L, BM) - g.t_first) * ceil_div(g.n_out, BN);
  if (tiles <= 0) return CASC_OK;
  // weight-resident: contiguous ranges; otherwise round-robin single tiles
  a.gt = WCH > 0 ? ceil_div(tiles, std::min<int64_t>(tiles, 148)) : 1;
  const int grid = (int)std::min<int64_t>(ceil_div(tiles, a.gt), 148);
  static unsigned long long* dbg = nullptr;
  const bool want_dbg = getenv("CASC_GEMM_DBG") != nullptr;
  if (want_dbg) {
    if (!dbg) CASC_TRY(cudaMalloc(&dbg, 24 * sizeof(unsigned long long)));
    CASC_TRY(cudaMemsetAsync(dbg, 0, 24 * sizeof(unsigned long long), st));
    a.dbg = dbg;
  }
  mimo_gemm_kernel<BN, TF32, RSO, WCH><<<grid, C::THREADS, C::SMEM, st>>>(maps, a);
  CASC_LAUNCHED();
  if (want_dbg) {                               // diagnostics only: synchronises and prints
    unsigned long long h[24];
    CASC_TRY(cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, st));
    CASC_TRY(cudaStreamSynchronize(st));
    static const char* nm[24] = {"prod.drain", "prod.empty", "", "", "mma.tempty", "mma.w_full", "mma.a_ready", "",
                                 "xf.full", "xf.alo_free", "", "", "epi.tfull", "epi.rfull", "", "", "", "", "", "",
                                 "res.rempty", "", "", "total"};
    const double tot = (double)h[23] / grid;
    fprintf(stderr, "casc gemm dbg BN=%d tf32=%d wch=%d n_src=%d grid=%d tiles=%lld: cycles/CTA %.0f |", BN, (int)TF32, WCH,
            g.n_src, grid, (long long)tiles, tot);
    for (int i = 0; i < 23; ++i)
      if (h[i]) fprintf(stderr, " %s %.0f%%", nm[i], 100.0 * h[i] / grid / tot / ((i == 8 || i == 9 || (i >= 12 && i < 16)) ? 4.0 : 1.0));
    fprintf(stderr, "\n");
  }
  return CASC_OK;
}

int launch_mimo_gemm(const MimoGemm& g, bool tf32, cudaStream_t st) {
  if (mimo_pair_ok(g, tf32)) return launch_mimo_gemm_pair(g, st);
  if (tf32 && mimo_pair_tf32_ok(g)) return launch_mimo_gemm_pair_tf32(g, st);
  if (g.peer_out) return CASC_ERR_UNSUPPORTED;      // peer-halo stores: CTA-pair kernels only
  // one-CTA kernel; template arguments <BN, TF32, residual/staging chunks, resident weight chunks>
  // are the measured-best splits of shared memory: 3xTF32 N = 64 keeps 4 residual
  // chunks (3 with the resident weights of a stage pair), bf16 N = 256 four (11% faster on E4 than 2)
  if (tf32) {
    if (g.n_out % 128 == 0) return launch_cfg<128, true>(g, st);   // main + corr accumulators
    if (g.n_out % 64 == 0) {
      if (g.w_resident) {                         // weights resident across tiles (bank stage)
        int chunks = 0;
        for (int s = 0; s < g.n_src; ++s) chunks += g.src[s].K / 32;
        if (chunks <= 2) return launch_cfg<64, true, 4, 2>(g, st);
        if (chunks <= 6) return launch_cfg<64, true, 3, 6>(g, st);
      }
      return launch_cfg<64, true>(g, st);
    }
  } else {
    if (g.n_out % 256 == 0) return launch_cfg<256, false, 4>(g, st);
    if (g.n_out % 128 == 0) return launch_cfg<128, false>(g, st);
    if (g.n_out % 64 == 0) return launch_cfg<64, false>(g, st);
  }
  return CASC_ERR_UNSUPPORTED;
}

}  // namespace casc
