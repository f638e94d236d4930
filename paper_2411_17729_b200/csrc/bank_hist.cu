// Bank streaming stage with the state history resident in shared memory (m = 64, 3xTF32).
//
// One pass applies (R23 in DESIGN.md)
//   v'(l) = v(l) + sum_{c=1..NS} W_c v(l - c s),   s = 2^k,
// NS = 1 (one stage, W_1 = P_k) or NS = 3 (stage pair, W = P_k, P_{k+1}, Q_k = P_{k+1} P_k).
// The multi-source GEMM (mimo_tc.cu) fetches every state tile 1 + NS times through L2 (as the
// residual of its own tile and as a shifted source of NS later tiles); on the pair pass that kept
// the L2 slices at ~91% of their measured throughput cap (profiles/). Here the tiles
// of a sequence are visited in residue-class order - with S = s / 128 tiles, the chain
// r, r + S, r + 2S, ... - so the sources of tile t = r + jS are the NS tiles visited just before
// it. Each tile is loaded once into a ring of four shared-memory slots and serves as the residual
// of its own output and as the A operand of the next NS tiles of its chain.
//
// Items. A CTA walks a contiguous range of positions (sequence, residue class, chain index j).
// Where a chain is entered at j > 0 (range start, or j0 = 1 for classes r < t_first) up to NS
// history-only "warm-up" items load the tiles t - cS >= 0 first. Item x lives in tile slot
// x % NSLOT and its tf32 split in TMEM history unit x % NH; the sources of compute item x are
// items x - 1 .. x - NS (sources with t - cS < 0 are zero and are skipped).
//
// Warps (10): 0 TMA producer (tiles + resident weights), 1 MMA issuer, 2-5 epilogue (TMEM
// accumulator + residual from the tile's slot -> 256-bit row stores of v', or the (C v, C P_Ne v)
// row parts, R24), 6-9 hi/lo split of each tile into its TMEM history unit.
// TMEM (512 columns): pair pass NS = 3: three history units of 128 columns (2 chunks x hi | lo)
// and one accumulator of 128 (main | corr); single pass NS = 1: two units, two accumulators.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "sm100.cuh"
#include "mimo_tc.cuh"
#include "profile.cuh"

namespace casc {
using namespace sm100;

namespace {
constexpr int HM = 64;                       // state dimension m
constexpr int HBM = 128;                     // rows per tile
constexpr uint32_t CHUNK = HBM * 128;        // one 32-column chunk of a tile: 16 KB
constexpr uint32_t SLOT = 2 * CHUNK;         // one tile (64 fp32 columns): 32 KB
constexpr uint32_t WCHUNK = HM * 128;        // one 32-column chunk of a weight (hi or lo): 8 KB
constexpr int THREADS = 10 * 32;
#ifndef HIST_SWAP
constexpr int PRODUCER_WARP = 0, MMA_WARP = 1;
#else
constexpr int PRODUCER_WARP = 1, MMA_WARP = 0;
#endif

__device__ __forceinline__ void h_tma_load(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void h_tma_store(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];"
               ::"l"(map), "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void h_named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void h_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void h_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
        "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
        "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

struct HistMaps {
  CUtensorMap V;      // source state [nseq][L][64] fp32, box {32, 128}
  CUtensorMap W[3];   // weight planes [planes][64][64] fp32 (tf32 hi / lo), box {32, 64}
};
struct HistArg {
  int ns;                               // shifted sources (1 or 3), shifts c * S tiles, c = 1..ns
  int S;                                // shift of source 1 in tiles (s / 128)
  int nt, t_first, nt_eff;              // tiles per sequence; first processed; processed per sequence
  int64_t L; int batch;
  const int* sys_list; int n_list;
  int w_plane_off[3], w_plane_stride[3];
  int64_t n_pos, gt;                    // positions in all, per CTA
  OutParts op;                          // fused output parts (R24-R26); planes == null: always store v
  float* out;                           // destination state [nseq][L][64]
  const int* tri;                       // per system: weights lower triangular (NEXT-3), or null
  unsigned long long* flops;            // issued tensor flops counter (profiling), or null
};

// One item of the CTA's walk: a compute tile or a history-only (warm-up) tile.
struct HItem {
  int seq, sys, t;
  bool compute;
};
struct HWalk {
  int64_t p, p_end;
  int w_left;                           // warm-up items still due before the compute item at p
  int seq, sys, r, j;                   // decoded position p
  int q, J, b, li;                      // position in its sequence, chain length, batch / list index
  __device__ void decode(const HistArg& a) {
    const int64_t si = p / a.nt_eff;
    q = (int)(p - si * a.nt_eff);
    J = a.nt / a.S;
    const int q0 = a.t_first * (J - 1);  // classes r < t_first start at j = 1 (tile r < t_first skipped)
    if (q < q0) { r = q / (J - 1); j = 1 + q % (J - 1); }
    else { const int q1 = q - q0; r = a.t_first + q1 / J; j = q1 % J; }
    li = (int)(si / a.batch); b = (int)(si % a.batch);
    sys = a.sys_list ? a.sys_list[li] : 0;
    seq = sys * a.batch + b;
  }
  __device__ HWalk(const HistArg& a) {
    p = (int64_t)blockIdx.x * a.gt;
    p_end = p + a.gt < a.n_pos ? p + a.gt : a.n_pos;
    if (p < p_end) { decode(a); w_left = j < a.ns ? j : a.ns; }
  }
  __device__ bool valid() const { return p < p_end; }
  __device__ HItem item(const HistArg& a) const {
    HItem it;
    it.seq = seq; it.sys = sys;
    it.compute = w_left == 0;
    it.t = r + (j - w_left) * a.S;
    return it;
  }
  // The walk advances one position at a time, so the decode is incremental: no integer division
  // and no channel-list load per item (the full decode of every item measured ~2.7k cycles of
  // the MMA warp's ~5.2k per item on E2: the issuing warp's loop bounded the pass).
  __device__ void next(const HistArg& a) {
    if (w_left > 0) { --w_left; return; }
    if (++p >= p_end) return;
    const int r0 = r, s0 = seq;
    if (++q == a.nt_eff) {                          // the next sequence
      q = 0;
      if (++b == a.batch) { b = 0; ++li; sys = a.sys_list ? a.sys_list[li] : 0; }
      seq = sys * a.batch + b;
      r = 0;
      j = a.t_first > 0 ? 1 : 0;
    } else {
      ++j;
    }
    while (j >= J) { ++r; j = r < a.t_first ? 1 : 0; }   // next class (classes r < t_first start at j = 1)
    // a new chain (class or sequence changed) is entered at its first processed tile j0 <= 1
    w_left = (r != r0 || seq != s0) ? (j < a.ns ? j : a.ns) : 0;
  }
};

// 256-bit global store (full 32-B sectors from one thread's row)
__device__ __forceinline__ void h_st8(float* p, const uint32_t* v) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]),
               "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
}

// NS = 3: three history units + one accumulator (512 TMEM columns), four shared-memory slots.
// NS = 1: two history units + two accumulators, six slots.
template <int NS>
struct HCfg {
  static constexpr int NH = NS == 3 ? 3 : 2;            // TMEM history units (128 columns: 2 chunks x hi | lo)
  static constexpr int NACC = NS == 3 ? 1 : 2;          // accumulators (128 columns: main | corr)
  static constexpr int NSLOT = NS == 3 ? 4 : 6;         // fp32 tile slots (32 KB)
  static constexpr uint32_t HB = NACC * 128;            // first history column
  static_assert(NACC * 128 + NH * 128 <= 512, "TMEM");
};

template <int NS>
__global__ void __launch_bounds__(THREADS, 1) bank_hist_kernel(const __grid_constant__ HistMaps maps, HistArg a) {
  using C = HCfg<NS>;
  constexpr int NH = C::NH, NACC = C::NACC, NSLOT = C::NSLOT;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sW = smem;                                   // [NS * 2 chunks][hi 8 KB | lo 8 KB]
  uint8_t* sT = smem + NS * 2 * 2 * WCHUNK;             // [NSLOT slots][2 chunks][16 KB]
  __shared__ uint64_t full[NSLOT], slot_free[NSLOT], hist_ready[NH], unit_free[NH], tfull[NACC], tempty[NACC], w_full,
      wfree;
  __shared__ uint32_t tmem_base;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const int S = a.S;

  if (threadIdx.x == 0) {
    // slot_free: the 128 split threads (tile read) and the 128 epilogue threads (residual read)
    for (int s = 0; s < NSLOT; ++s) { mbar_init(&full[s], 1); mbar_init(&slot_free[s], 256); }
    for (int u = 0; u < NH; ++u) { mbar_init(&hist_ready[u], 128); mbar_init(&unit_free[u], 1); }
    for (int c = 0; c < NACC; ++c) { mbar_init(&tfull[c], 1); mbar_init(&tempty[c], 128); }
    mbar_init(&w_full, 1);
    mbar_init(&wfree, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tmem_base != 0) __trap();                         // 512 columns: the whole TMEM, base 0

  if (warp == PRODUCER_WARP) {
    // =========================================================== TMA producer (whole warp loops)
    const bool issue = lane == 0;
    int cur_sys = -1, n_reload = 0;
    int64_t x = 0;
    for (HWalk w(a); w.valid(); w.next(a), ++x) {
      const HItem it = w.item(a);
      if (it.compute && it.sys != cur_sys) {
        if (n_reload > 0) mbar_wait(&wfree, (uint32_t)((n_reload - 1) & 1));
        ++n_reload;
        if (issue) {
          mbar_arrive_expect_tx(&w_full, NS * 2 * 2 * WCHUNK);
          for (int c = 0; c < NS; ++c) {
            const int plane = it.sys * a.w_plane_stride[c] + a.w_plane_off[c];
            for (int kc = 0; kc < 2; ++kc) {
              uint8_t* dst = sW + (c * 2 + kc) * 2 * WCHUNK;
              h_tma_load(dst, &maps.W[c], &w_full, kc * 32, 0, plane);
              h_tma_load(dst + WCHUNK, &maps.W[c], &w_full, kc * 32, 0, plane + 1);
            }
          }
        }
        cur_sys = it.sys;
      }
      const int s = (int)(x % NSLOT);
      if (x >= NSLOT) mbar_wait(&slot_free[s], (uint32_t)((x / NSLOT - 1) & 1));   // item x - NSLOT is done
      if (issue) {
        mbar_arrive_expect_tx(&full[s], SLOT);
        uint8_t* dst = sT + s * SLOT;
        h_tma_load(dst, &maps.V, &full[s], 0, it.t * HBM, it.seq);
        h_tma_load(dst + CHUNK, &maps.V, &full[s], 32, it.t * HBM, it.seq);
      }
    }
  } else if (warp == MMA_WARP) {
    // =========================================================== MMA issuer (whole warp, elected lane)
    const uint32_t idesc = make_idesc(FMT_TF32, HBM, HM), idesc128 = make_idesc(FMT_TF32, HBM, 2 * HM);
    int cur_sys = -1;
    bool lower = false;                              // this system's weights are lower triangular
    unsigned n_tri = 0, n_dense = 0;                 // sources issued with / without the triangular skip
    uint32_t wph = 0;
    int64_t z = 0, tl = 0;
    for (HWalk w(a); w.valid(); w.next(a), ++z) {
      const HItem it = w.item(a);
      // Release the unit of item y = z - NS (no MMA after this item reads it). Its split must have
      // landed first even when no MMA read it: the transform writing the unit next waits for this
      // release by phase parity, so releases may not run ahead of the splits they release.
      auto release = [&](bool waited) {
        if (z < NS) return;
        const int64_t y = z - NS;
        if (!waited) mbar_wait_u(&hist_ready[(int)(y % NH)], (uint32_t)((y / NH) & 1));
        mma_commit_w(&unit_free[(int)(y % NH)]);
      };
      if (!it.compute) {                              // history only
        release(false);
        continue;
      }
      if (it.sys != cur_sys) {
        if (cur_sys >= 0) mma_commit_w(&wfree);       // every MMA so far used the previous weights
        mbar_wait_u(&w_full, wph);
        wph ^= 1;
        cur_sys = it.sys;
        // warp-uniform (broadcast from lane 0): the MMA branch below must not diverge
        lower = __shfl_sync(0xffffffffu, a.tri ? a.tri[it.sys] : 0, 0) != 0;
      }
      const int acc = (int)(tl % NACC);
      mbar_wait_u(&tempty[acc], (uint32_t)(((tl / NACC) & 1) ^ 1));
      tc_fence_after();
      const uint32_t d = acc * 128, dc = d + HM;
      // the tile's MMAs, instantiated once per weight structure so neither path carries the other's
      // branches (the issuing warp's instruction stream bounds this kernel)
      auto issue = [&](auto tri_tag) {
        constexpr bool TRI = decltype(tri_tag)::value;
        bool first = true;
#pragma unroll
        for (int c = NS; c >= 1; --c) {               // oldest source first: its unit is freed early
          const int64_t y = z - c;                    // the source item
          if (it.t >= c * S) {
            const int u = (int)(y % NH);
            mbar_wait_u(&hist_ready[u], (uint32_t)((y / NH) & 1));
            tc_fence_after();
#pragma unroll
            for (int kc = 0; kc < 2; ++kc) {
              const uint32_t ah = C::HB + (uint32_t)u * 128 + kc * 64, al = ah + 32;
              const uint64_t wd = make_sdesc(smem_u32(sW + ((c - 1) * 2 + kc) * 2 * WCHUNK), 16, 1024, LAYOUT_SW128);
              if constexpr (TRI) {                    // NEXT-3: skip the all-zero upper blocks
                if (kc == 0) mma_3xtf32_ts_chunk8_tri_w<0>(d, dc, ah, al, wd, first ? 0u : 1u);
                else mma_3xtf32_ts_chunk8_tri_w<1>(d, dc, ah, al, wd, first ? 0u : 1u);
              } else {
                mma_3xtf32_ts_chunk8_w(d, dc, ah, al, wd, idesc128, idesc, first ? 0u : 1u);
              }
              first = false;
            }
            if constexpr (TRI) ++n_tri; else ++n_dense;
          }
          // the unit of item z - NS is read last by these (source c = NS) MMAs
          if (c == NS) release(it.t >= NS * S);
        }
      };
      if (lower) issue(std::true_type{});
      else issue(std::false_type{});
      mma_commit_w(&tfull[acc]);
      ++tl;
    }
    // issued flops (profiling): N-columns x K-steps per source, each worth 2 * 128 * 8 flops (M = 128, K = 8)
    if (a.flops && lane == 0) {
      const unsigned long long cols = (unsigned long long)n_tri * (tri_chunk_cols<0>() + tri_chunk_cols<1>()) +
                                      (unsigned long long)n_dense * 2 * 4 * (2 * HM + HM);
      atomicAdd(a.flops, cols * (unsigned long long)(2 * HBM * 8));
    }
  } else if (warp >= 6) {
    // =========================================================== split every tile once into its TMEM unit
    const int row = (warp & 3) * 32 + lane;
    const uint32_t lanes = (uint32_t)((warp & 3) * 32) << 16;
    int64_t x = 0;
    for (HWalk w(a); w.valid(); w.next(a), ++x) {
      const int s = (int)(x % NSLOT), u = (int)(x % NH);
      mbar_wait(&full[s], (uint32_t)((x / NSLOT) & 1));
      uint32_t hv[64], lv[64];
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) {
        const uint8_t* rr = sT + s * SLOT + kc * CHUNK + row * 128;     // SW128: 16-B chunk cc at (cc ^ row % 8)
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const float4 v = *reinterpret_cast<const float4*>(rr + ((cc ^ (row & 7)) * 16));
          const float4 h = tf32_hi4(v), l = tf32_lo4(v, h);
          const int o = kc * 32 + 4 * cc;
          hv[o] = __float_as_uint(h.x); hv[o + 1] = __float_as_uint(h.y);
          hv[o + 2] = __float_as_uint(h.z); hv[o + 3] = __float_as_uint(h.w);
          lv[o] = __float_as_uint(l.x); lv[o + 1] = __float_as_uint(l.y);
          lv[o + 2] = __float_as_uint(l.z); lv[o + 3] = __float_as_uint(l.w);
        }
      }
      mbar_arrive(&slot_free[s]);                     // tile read
      if (x >= NH) mbar_wait_u(&unit_free[u], (uint32_t)((x / NH - 1) & 1));   // unit of item x - NH released
      tc_fence_after();
      const uint32_t ta = lanes + C::HB + (uint32_t)u * 128;
      h_st32(ta, hv);
      h_st32(ta + 32, lv);
      h_st32(ta + 64, hv + 32);
      h_st32(ta + 96, lv + 32);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      mbar_arrive(&hist_ready[u]);
    }
  } else {
    // =========================================================== epilogue (warps 2..5): row per thread
    const int q = warp & 3;
    const int row = q * 32 + lane;
    int64_t x = 0, tl = 0;
    for (HWalk w(a); w.valid(); w.next(a), ++x) {
      const HItem it = w.item(a);
      const int sr = (int)(x % NSLOT);
      if (!it.compute) {                              // history only: no residual read
        // arrive only once the item has landed: its load waited for the slot's previous phase to
        // complete, so this arrival cannot count towards the previous occupant's release
        mbar_wait(&full[sr], (uint32_t)((x / NSLOT) & 1));
        mbar_arrive(&slot_free[sr]);
        continue;
      }
      const int acc = (int)(tl % NACC);
      int depth = 0;                                  // this channel's parts at this level, if any
      bool to_parts = false;
      if (a.op.planes != nullptr) {
        const int ne = a.op.neff[it.sys];
        depth = fold_depth(ne, a.op.kc[it.sys], a.op.fold);
        to_parts = ne - depth == a.op.level;
      }
      const bool any_src = it.t >= S;
      // warp-uniform waits before the .sync.aligned tcgen05.ld / st: a per-lane spin loop can
      // leave the warp diverged there (measured: one 32-row quadrant of a tile corrupted)
      mbar_wait_u(&tfull[acc], (uint32_t)((tl / NACC) & 1));
      tc_fence_after();
      uint32_t vm[64], vc[64];
      if (any_src) {
        const uint32_t ta = ((uint32_t)(q * 32) << 16) + acc * 128;
        h_ld32(ta, vm);
        h_ld32(ta + 32, vm + 32);
        h_ld32(ta + HM, vc);
        h_ld32(ta + HM + 32, vc + 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      } else {
#pragma unroll
        for (int e = 0; e < 64; ++e) vm[e] = vc[e] = 0u;
      }
      mbar_wait(&full[sr], (uint32_t)((x / NSLOT) & 1));   // this tile (the residual) has landed
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) {
        const uint8_t* rrow = sT + sr * SLOT + kc * CHUNK + row * 128;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const float4 r = *reinterpret_cast<const float4*>(rrow + (cc ^ (row & 7)) * 16);
          const int col = kc * 32 + cc * 4;
          vm[col] = __float_as_uint(r.x + (__uint_as_float(vm[col]) + __uint_as_float(vc[col])));
          vm[col + 1] = __float_as_uint(r.y + (__uint_as_float(vm[col + 1]) + __uint_as_float(vc[col + 1])));
          vm[col + 2] = __float_as_uint(r.z + (__uint_as_float(vm[col + 2]) + __uint_as_float(vc[col + 2])));
          vm[col + 3] = __float_as_uint(r.w + (__uint_as_float(vm[col + 3]) + __uint_as_float(vc[col + 3])));
        }
      }
      // Release the accumulator only now: tcgen05.wait::ld orders nothing but later uses of the
      // loaded registers (SASS has no wait instruction; the register scoreboard does it), so an
      // arrive placed before the first use let the next tile's MMA overwrite TMEM under a lagging warp.
      tc_fence_before();
      mbar_arrive(&tempty[acc]);                      // accumulator drained (every loaded value used)
      mbar_arrive(&slot_free[sr]);                    // residual rows read
      const int64_t l = (int64_t)it.t * HBM + row;
      if (to_parts) {                                 // the 2^(depth+1) output parts of this row
        const float* vb = a.op.vec + (int64_t)it.sys * kMaxParts * HM;
        const int np = 2 << depth;
        const int64_t r = (int64_t)it.seq * a.L + l;
        for (int b = 0; b < np; ++b) {
          float p = 0.f;
#pragma unroll
          for (int col = 0; col < HM; col += 4) {
            const float4 c4 = __ldg(reinterpret_cast<const float4*>(vb + b * HM + col));
            p = fmaf(c4.x, __uint_as_float(vm[col]), p); p = fmaf(c4.y, __uint_as_float(vm[col + 1]), p);
            p = fmaf(c4.z, __uint_as_float(vm[col + 2]), p); p = fmaf(c4.w, __uint_as_float(vm[col + 3]), p);
          }
          if (l < a.L) a.op.planes[b * a.op.plane + r] = p;
        }
      } else if (l < a.L) {
        float* orow = a.out + ((int64_t)it.seq * a.L + l) * HM;
#pragma unroll
        for (int e = 0; e < 8; ++e) h_st8(orow + 8 * e, vm + 8 * e);
      }
      ++tl;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(0);
}
}  // namespace

// Applicable to the bank stage passes: fp32, m = 64, 1 or 3 sources A = R = v at shifts c * s,
// s a multiple of 128 with the tile count a multiple of s / 128, no halo rows.
static char hist_mode() {     // CASC_BANK_HIST = 0 (off) | p (stage pairs only) | s (single stages only)
  static const char mode = [] {
    const char* e = getenv("CASC_BANK_HIST");
    return e ? e[0] : '1';
  }();
  return mode;
}
bool bank_hist_ok(int64_t L, int64_t shift, int n_src, int t_first) {
  const char mode = hist_mode();
  if (mode == '0' || (mode == 'p' && n_src != 3) || (mode == 's' && n_src != 1)) return false;
  if (!(n_src == 1 || n_src == 3) || shift <= 0 || shift % HBM) return false;
  const int nt = (int)((L + HBM - 1) / HBM), S = (int)(shift / HBM);
  if (S > nt || nt % S || (t_first >= S && t_first > 0)) return false;
  return !(nt / S == 1 && t_first > 0);
}
int launch_bank_hist(const MimoGemm& g, cudaStream_t st) {
  const char mode = hist_mode();
  if (mode == '0' || (mode == 'p' && g.n_src != 3) || (mode == 's' && g.n_src != 1)) return CASC_ERR_UNSUPPORTED;
  if (g.n_out != HM || !(g.n_src == 1 || g.n_src == 3) || g.R_row0 || g.out_row0) return CASC_ERR_UNSUPPORTED;
  const int64_t s = g.src[0].shift;
  if (s <= 0 || s % HBM) return CASC_ERR_UNSUPPORTED;
  for (int c = 0; c < g.n_src; ++c)
    if (g.src[c].K != HM || g.src[c].A != g.R || g.src[c].shift != (c + 1) * s || g.src[c].row0) return CASC_ERR_UNSUPPORTED;
  const int nt = (int)((g.L + HBM - 1) / HBM), S = (int)(s / HBM);
  if (S > nt || nt % S || g.t_first >= S && g.t_first > 0) return CASC_ERR_UNSUPPORTED;
  if (nt / S == 1 && g.t_first > 0) return CASC_ERR_UNSUPPORTED;
  HistMaps maps;
  memset(&maps, 0, sizeof(maps));
  HistArg a{};
  a.ns = g.n_src; a.S = S; a.nt = nt; a.t_first = g.t_first; a.nt_eff = nt - g.t_first;
  a.L = g.L; a.batch = g.batch; a.sys_list = g.sys_list; a.n_list = g.sys_list ? g.n_list : 1;
  a.op = g.parts;
  a.tri = g.tri;
  a.flops = g.flop_counter;
  const int64_t nseq_total = (int64_t)(g.n_sys_total > 0 ? g.n_sys_total : 1) * g.batch;
  if (!map3d(&maps.V, g.R, true, HM, g.L, nseq_total, HBM)) return CASC_ERR_CUDA;
  a.out = static_cast<float*>(g.out);
  for (int c = 0; c < g.n_src; ++c) {
    a.w_plane_off[c] = g.src[c].w_plane_off;
    a.w_plane_stride[c] = g.src[c].w_plane_stride;
    const int64_t planes = g.src[c].w_planes > 0 ? g.src[c].w_planes : 2;
    if (!map3d(&maps.W[c], g.src[c].W, true, HM, HM, planes, HM)) return CASC_ERR_CUDA;
  }
  a.n_pos = (int64_t)a.n_list * g.batch * a.nt_eff;
  if (a.n_pos == 0) return CASC_OK;
  const int grid = (int)std::min<int64_t>(a.n_pos, 148);
  a.gt = (a.n_pos + grid - 1) / grid;
  const int grid_used = (int)((a.n_pos + a.gt - 1) / a.gt);
  // pairs: 96 KB of weights + 4 slots; single stages: 32 KB + 6 slots (loads run further ahead)
  if (g.n_src == 3) {
    const size_t smem = 1024 + (size_t)3 * 2 * 2 * WCHUNK + (size_t)HCfg<3>::NSLOT * SLOT;
    if (cudaFuncSetAttribute(bank_hist_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return CASC_ERR_CUDA;
    bank_hist_kernel<3><<<grid_used, THREADS, smem, st>>>(maps, a);
  } else {
    const size_t smem = 1024 + (size_t)1 * 2 * 2 * WCHUNK + (size_t)HCfg<1>::NSLOT * SLOT;
    if (cudaFuncSetAttribute(bank_hist_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return CASC_ERR_CUDA;
    bank_hist_kernel<1><<<grid_used, THREADS, smem, st>>>(maps, a);
  }
  CASC_LAUNCHED();
  return cudaGetLastError() == cudaSuccess ? CASC_OK : CASC_ERR_CUDA;
}

}  // namespace casc
