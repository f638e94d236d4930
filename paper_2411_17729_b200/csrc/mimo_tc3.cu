// Shifted multi-source GEMM, 3xTF32, on CTA PAIRS (tcgen05 cta_group::2): the fp32 MIMO steps
// with 128-column output blocks (E3: m = 256) of PAPER.md:185-229, the same map as mimo_tc.cu
//   out[s][l][n] = sum_src sum_k A_src[s][l - shift_src][k] W_src[n][k]  (+ R[s][l][n])
// One-CTA tiles re-read the 128 x K tf32 hi/lo weights through L2 for every 128 rows: on E3 that
// was 4.2 of the 10.1 GB of L2 traffic per stage, and the L2 slices bounded the kernel.
// Here a cluster of two CTAs computes 256 x 128 tiles: each CTA stages its 128 rows of A and 64 of
// the 128 weight rows, and the leader issues M = 256, N = 128, K = 8 MMAs that read both CTAs'
// shared memory, so every CTA moves half the weight bytes per K chunk.
//
// 3xTF32 as in mimo_tc.cu: hi.hi into the main accumulator, lo.hi + hi.lo into the correction
// accumulator (separate truncation chains), summed with round-to-nearest in the epilogue. Four
// transform warps per CTA write the lo part of the landed A chunk (lo = rna(v - trunc_tf32(v)); the
// MMA reads the raw chunk as hi, truncated by the tensor core).
//
// Protocol: A lands on a CTA-local barrier (its transform waits for it); both CTAs' weight loads
// and both CTAs' transforms signal barriers in the LEADER (the weight loads through the 2-SM TMA
// form, the transforms by remote arrive); MMA completion is multicast to both CTAs' ring-slot and
// accumulator-full barriers; both CTAs' epilogues release the accumulator on the leader's barrier.
// TMEM: 2 accumulators x (128 main | 128 corr) = 512 columns per CTA, allocated with cta_group::2.
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>

#include "common.cuh"
#include "sm100.cuh"
#include "mimo_tc.cuh"

namespace casc {
using namespace sm100;

namespace {
constexpr int HM = 128;                   // rows per CTA
constexpr int BK = 32;                    // fp32 K per chunk (128-byte rows)
constexpr uint32_t A_BYTES = HM * 128;    // 16 KB (hi in place; lo in its own 16 KB)
// residual / staging chunks (128 rows x 32 fp32): four, so the residual loads of a tile's chunks run
// ahead of the epilogue (their HBM latency paced it with two: 4.3k cycles of waits per tile); paid
// for with one ring stage (3 instead of 4). E3 A/B (forced rebuilds): 9.40 -> 9.02 ms min.
constexpr int RS = 4;
constexpr uint32_t R_BYTES = HM * 128;
constexpr int CW = 32;                    // epilogue chunk width (fp32 columns = 128 bytes)
constexpr int THREADS = 11 * 32;          // 0 TMA, 1 MMA, 2-5 epilogue, 6-9 transform, 10 residual
// BN output columns per pair tile: 128 (two TMEM accumulators, 3 ring slots + 4 residual chunks)
// SPLIT: main (hi.hi) accumulators per tile. The tensor core truncates its fp32 accumulator at every
// MMA, so the main chain's error grows with K / 8; long contractions (K > 512) spread
// the main chain over SPLIT = 3 accumulators (one third of the K chunks each, summed with
// round-to-nearest in the epilogue), at the price of a single accumulator set (SPLIT mains + corr =
// 4 x 128 = 512 TMEM columns, no double buffering).
template <int BN, int SPLIT = 1>
struct PCfg {
  static constexpr uint32_t W_BYTES = (BN / 2) * 128;             // this CTA's BN/2 weight rows, hi or lo
  static constexpr uint32_t STAGE_BYTES = 2 * A_BYTES + 2 * W_BYTES;   // A hi | A lo | W hi | W lo
  static constexpr int STAGES = 3;
  static constexpr int NACC = (BN == 256 || SPLIT > 1) ? 1 : 2;
  static constexpr uint32_t ACC_COLS = (SPLIT + 1) * BN;           // SPLIT mains | corr
  static_assert(NACC * ACC_COLS <= 512, "TMEM");
  static constexpr int NCH = BN / CW;
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + RS * R_BYTES;
};

__device__ __forceinline__ uint32_t cta_rank3() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync3() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2sm3(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_load_13(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];"
               ::"l"(map), "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void named_sync3(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void mma_tf32_pair_w(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// The same MMA keeping its A operand in the tensor core's collector buffer (fill) / reading it from
// there and releasing it (lastuse): the two products of a K step that share A_hi (hi.hi, hi.lo)
// read A_hi from shared memory once (SASS UTCHMMA .A_KEEP / .A_REUSE). E3: 9.02 -> 8.80 ms min.
__device__ __forceinline__ void mma_tf32_pair_fill_w(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::2.kind::tf32.collector::a::fill [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_tf32_pair_lastuse_w(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::2.kind::tf32.collector::a::lastuse [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_pair3(uint64_t* bar) {   // both CTAs' barrier at this offset
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
__device__ __forceinline__ void arrive_leader3(uint64_t* bar) {    // arrive on the leader CTA's copy
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  // default semantics (release, CTA scope), as for a local arrive: the writes this orders are
  // the arriving thread's own shared-memory stores, already fenced to the async proxy
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void tmem_ld32_3(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

struct PairCoord3 {
  int seq, l0, nb;     // l0: first row of this CTA's half
};
template <int BN>
__device__ __forceinline__ PairCoord3 decode3(int64_t tile, const MimoArg& a, int n_nblk, int64_t nb_eff, int t0_blk,
                                              uint32_t rank) {
  PairCoord3 t;
  t.nb = (int)(tile % n_nblk);
  const int64_t r = tile / n_nblk;
  t.l0 = (int)((t0_blk + r % nb_eff) * (2 * HM) + rank * HM);
  t.seq = (int)(r / nb_eff);                      // one system: sequence = batch index
  return t;
}
}  // namespace

template <int BN, int SPLIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    mimo_gemm_pair_tf32_kernel(const __grid_constant__ MimoMaps maps, MimoArg a) {
  using C = PCfg<BN, SPLIT>;
  constexpr int STAGES = C::STAGES, NACC = C::NACC, NCH = C::NCH;
  constexpr uint32_t STAGE_BYTES = C::STAGE_BYTES, W_BYTES = C::W_BYTES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sR = smem + STAGES * STAGE_BYTES;
  __shared__ uint64_t full_a[STAGES], full_w[STAGES], lo_ready[STAGES], empty[STAGES], tfull[NACC], tempty[NACC], rfull[RS],
      rempty[RS];
  __shared__ uint32_t tmem_base;
  auto stA = [&](int s) { return smem + s * STAGE_BYTES; };
  auto stAlo = [&](int s) { return smem + s * STAGE_BYTES + A_BYTES; };
  auto stW = [&](int s) { return smem + s * STAGE_BYTES + 2 * A_BYTES; };   // hi, then lo at + W_BYTES

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const uint32_t rank = cta_rank3();
  const bool is_leader = rank == 0;
  const int64_t blocks_per_b = (a.L + 2 * HM - 1) / (2 * HM);
  const int t0_blk = a.t_first / 2;
  const int64_t nb_eff = blocks_per_b - t0_blk;
  const int n_nblk = (a.n_out + BN - 1) / BN;
  const int64_t n_tiles = (int64_t)a.batch * nb_eff * n_nblk;
  const int64_t pair = blockIdx.x / 2, n_pairs = gridDim.x / 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_a[s], 1); mbar_init(&full_w[s], 1); mbar_init(&lo_ready[s], 2 * 128); mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < NACC; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 2 * 128); }
    for (int s = 0; s < RS; ++s) { mbar_init(&rfull[s], 1); mbar_init(&rempty[s], 1); }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync3();                                         // both CTAs' barriers and TMEM ready
  tc_fence_after();
  if (tmem_base != 0) __trap();                            // 512 columns: the whole TMEM
  constexpr uint32_t tbase = 0;

  if (warp == 0) {
    // =========================================================== TMA producer (both CTAs, whole warp loops)
    const bool issue = lane == 0;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = pair; t < n_tiles; t += n_pairs) {
      const PairCoord3 tc = decode3<BN>(pair_tile_order(t, n_pairs, n_nblk, n_tiles), a, n_nblk, nb_eff, t0_blk, rank);
      for (int src = 0; src < a.n_src; ++src) {
        const int nk = a.K[src] / BK;
        const int plane = a.w_plane_off[src];
        for (int kc = 0; kc < nk; ++kc) {
          mbar_wait(&empty[s], ph ^ 1);
          if (issue) {
            mbar_arrive_expect_tx(&full_a[s], A_BYTES);   // this CTA's rows of A: local barrier
            tma_load_13(stA(s), &maps.A[src], &full_a[s], kc * BK, a.a_row0[src] + tc.l0 - (int)a.shift[src], tc.seq);
            if (is_leader) mbar_arrive_expect_tx(&full_w[s], 2 * 2 * W_BYTES);   // both CTAs' W hi + lo
            uint32_t fw;                          // the leader CTA's full_w[s] (shared::cluster)
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(fw) : "r"(smem_u32(&full_w[s])));
            tma_load_2sm3(stW(s), &maps.W[src], fw, kc * BK, tc.nb * BN + (int)rank * (BN / 2), plane);
            tma_load_2sm3(stW(s) + W_BYTES, &maps.W[src], fw, kc * BK, tc.nb * BN + (int)rank * (BN / 2), plane + 1);
          }
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 10) {
    // =========================================================== residual / staging producer (per CTA)
    const bool issue = lane == 0;
    int rs = 0;
    uint32_t rph = 0;
    for (int64_t t = pair; t < n_tiles; t += n_pairs) {
      const PairCoord3 tc = decode3<BN>(pair_tile_order(t, n_pairs, n_nblk, n_tiles), a, n_nblk, nb_eff, t0_blk, rank);
      for (int j = 0; j < NCH; ++j) {
        mbar_wait(&rempty[rs], rph ^ 1);
        if (!issue) {
        } else if (a.has_residual) {
          mbar_arrive_expect_tx(&rfull[rs], R_BYTES);
          tma_load_13(sR + rs * R_BYTES, &maps.R, &rfull[rs], tc.nb * BN + j * CW, a.r_row0 + tc.l0, tc.seq);
        } else {
          mbar_arrive(&rfull[rs]);
        }
        if (++rs == RS) { rs = 0; rph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // =========================================================== MMA issuer (leader CTA, whole warp)
    if (is_leader) {
      const uint32_t idesc = make_idesc(FMT_TF32, 2 * HM, BN);
      int s = 0;
      uint32_t ph = 0;
      int64_t t_local = 0;
      for (int64_t t = pair; t < n_tiles; t += n_pairs, ++t_local) {
        const int acc = (int)(t_local % NACC);
        mbar_wait_u(&tempty[acc], (uint32_t)((t_local / NACC) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d0 = tbase + acc * C::ACC_COLS, dc = d0 + SPLIT * BN;
        int nk_all = 0;
        for (int src = 0; src < a.n_src; ++src) nk_all += a.K[src] / BK;
        bool fm[SPLIT], fc = true;                    // first write of each main / of the correction
#pragma unroll
        for (int i = 0; i < SPLIT; ++i) fm[i] = true;
        int j = 0;                                    // K chunk of the tile, all sources in order
        for (int src = 0; src < a.n_src; ++src) {
          const int nk = a.K[src] / BK;
          for (int kc = 0; kc < nk; ++kc, ++j) {
            const int mi = SPLIT > 1 ? j * SPLIT / nk_all : 0;   // this chunk's main accumulator
            const uint32_t d = d0 + mi * BN;
            mbar_wait_u(&full_w[s], ph);
            mbar_wait_u(&lo_ready[s], ph);
            tc_fence_after();
            const uint64_t ad0 = make_sdesc(smem_u32(stA(s)), 16, 1024, LAYOUT_SW128);
            const uint64_t al0 = make_sdesc(smem_u32(stAlo(s)), 16, 1024, LAYOUT_SW128);
            const uint64_t wd0 = make_sdesc(smem_u32(stW(s)), 16, 1024, LAYOUT_SW128);
            const uint64_t wl0 = make_sdesc(smem_u32(stW(s) + W_BYTES), 16, 1024, LAYOUT_SW128);
            bool first_m = false;
#pragma unroll
            for (int i = 0; i < SPLIT; ++i)
              if (i == mi) { first_m = fm[i]; fm[i] = false; }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t ad = sdesc_add(ad0, k * 32), wd = sdesc_add(wd0, k * 32);
              mma_tf32_pair_fill_w(d, ad, wd, idesc, (first_m && k == 0) ? 0u : 1u);      // main: hi.hi (A_hi kept)
              mma_tf32_pair_lastuse_w(dc, ad, sdesc_add(wl0, k * 32), idesc, (fc && k == 0) ? 0u : 1u);  // corr: hi.lo
              mma_tf32_pair_w(dc, sdesc_add(al0, k * 32), wd, idesc, 1u);                //     + lo.hi
            }
            fc = false;
            mma_commit_pair3(&empty[s]);
            if (++s == STAGES) { s = 0; ph ^= 1; }
          }
        }
        mma_commit_pair3(&tfull[acc]);
      }
    }
  } else if (warp >= 6) {
    // =========================================================== hi/lo split of the landed A chunk (per CTA)
    const int t = threadIdx.x - 192;             // 0..127: one 128-byte row each
    int s = 0;
    uint32_t ph = 0;
    for (int64_t tt = pair; tt < n_tiles; tt += n_pairs) {
      for (int src = 0; src < a.n_src; ++src) {
        const int nk = a.K[src] / BK;
        for (int kc = 0; kc < nk; ++kc) {
          mbar_wait(&full_a[s], ph);
          float4* hi = reinterpret_cast<float4*>(stA(s));
          float4* lo = reinterpret_cast<float4*>(stAlo(s));
#pragma unroll
          for (int e = t; e < (int)(A_BYTES / 16); e += 128) {   // the swizzle is the same for hi and lo
            // hi stays the raw chunk (the MMA reads its tf32 truncation); only lo is written: one
            // shared-memory store stream less per chunk (E3 8.80 -> 8.36 ms min, same accuracy)
            const float4 v = hi[e];
            lo[e] = tf32_lo4(v, tf32_trunc4(v));
          }
          fence_async_smem();                    // generic writes -> the MMA's async proxy
          if (is_leader) mbar_arrive(&lo_ready[s]);
          else arrive_leader3(&lo_ready[s]);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else {
    // =========================================================== epilogue (warps 2..5, both CTAs)
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const bool leader_t = (warp == 2 && lane == 0);
    int64_t t_local = 0;
    int rs = 0, prev_rs = -1;
    uint32_t rph = 0;
    for (int64_t t = pair; t < n_tiles; t += n_pairs, ++t_local) {
      const PairCoord3 tc = decode3<BN>(pair_tile_order(t, n_pairs, n_nblk, n_tiles), a, n_nblk, nb_eff, t0_blk, rank);
      const int acc = (int)(t_local % NACC);
      mbar_wait_u(&tfull[acc], (uint32_t)((t_local / NACC) & 1));
      tc_fence_after();
      for (int j = 0; j < NCH; ++j) {
        uint8_t* rbuf = sR + rs * R_BYTES;
        uint32_t vm[32], vc[32];
        const uint32_t taddr = tbase + ((uint32_t)(q * 32) << 16) + acc * C::ACC_COLS + j * CW;
        float f[32];
        if constexpr (SPLIT == 1) {
          tmem_ld32_3(taddr, vm);
          tmem_ld32_3(taddr + BN, vc);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int e = 0; e < 32; ++e) f[e] = __uint_as_float(vm[e]) + __uint_as_float(vc[e]);   // main + corr
        } else {                                      // ((main_0 + main_1) + ...) + corr, round-to-nearest
          tmem_ld32_3(taddr, vm);
          tmem_ld32_3(taddr + SPLIT * BN, vc);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int e = 0; e < 32; ++e) f[e] = __uint_as_float(vm[e]);
#pragma unroll
          for (int i = 1; i < SPLIT; ++i) {
            tmem_ld32_3(taddr + i * BN, vm);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int e = 0; e < 32; ++e) f[e] += __uint_as_float(vm[e]);
          }
#pragma unroll
          for (int e = 0; e < 32; ++e) f[e] += __uint_as_float(vc[e]);
        }
        if (j == NCH - 1) {                       // accumulator drained (values consumed): release it
          tc_fence_before();
          if (is_leader) mbar_arrive(&tempty[acc]);
          else arrive_leader3(&tempty[acc]);
        }
        mbar_wait(&rfull[rs], rph);
        uint8_t* rrow = rbuf + row * 128;         // SW128: 16-B chunk c at ((c ^ (row % 8)) * 16)
        // the successor rank's halo rows (peer halo, seqshard.cu), from registers over the peer mapping
        const int64_t lrow = (int64_t)tc.l0 + row;
        float* prow = (a.peer_out && lrow >= a.peer_l_begin && lrow < a.L)
            ? static_cast<float*>(a.peer_out) + ((int64_t)tc.seq * (a.out_row0 + a.L) + a.out_row0 + lrow - a.peer_shift) * a.n_out + tc.nb * BN + j * CW
            : nullptr;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float4* p = reinterpret_cast<float4*>(rrow + ((c ^ (row & 7)) * 16));
          float4 o = make_float4(f[4 * c], f[4 * c + 1], f[4 * c + 2], f[4 * c + 3]);
          if (a.has_residual) {
            const float4 r = *p;
            o.x += r.x; o.y += r.y; o.z += r.z; o.w += r.w;
          }
          *p = o;
          if (prow) *reinterpret_cast<float4*>(prow + 4 * c) = o;
        }
        fence_async_smem();
        named_sync3(1, 128);
        if (leader_t) {
          tma_store3(&maps.out, rbuf, tc.nb * BN + j * CW, a.out_row0 + tc.l0, tc.seq);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          if (prev_rs >= 0) {                     // the previous chunk's store has read its slot
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            mbar_arrive(&rempty[prev_rs]);
          }
        }
        prev_rs = rs;
        if (++rs == RS) { rs = 0; rph ^= 1; }
      }
    }
    if (leader_t) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (a.peer_out) __threadfence_system();       // peer stores visible before the kernel completes
  }
  tc_fence_before();
  cluster_sync3();                                         // no CTA of the pair still uses TMEM
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512) : "memory");
}

bool mimo_pair_tf32_ok(const MimoGemm& g) {
  static const bool off = [] {
    const char* e = getenv("CASC_GEMM_PAIR_TF32");
    return e && e[0] == '0';
  }();
  // 128-wide tiles (64-wide outputs stay on the one-CTA kernel: the E3 output stage measured 0.47
  // ms there vs 0.59 ms on pairs; a 256-wide tile with one accumulator measured 0.87 vs 0.81 ms)
  if (off || g.n_out % 128 != 0 || g.w_resident || g.ab || g.parts_deep || g.sys_list != nullptr) return false;
  for (int s = 0; s < g.n_src; ++s)
    if (g.src[s].K % BK || g.src[s].w_plane_stride != 0) return false;   // one weight plane pair per source
  return true;
}

template <int BN, int SPLIT>
static int launch_pt(const MimoGemm& g, cudaStream_t st) {
  using C = PCfg<BN, SPLIT>;
  MimoMaps maps;
  memset(&maps, 0, sizeof(maps));
  MimoArg a{};
  a.n_src = g.n_src;
  a.L = g.L;
  a.batch = g.batch;
  a.n_out = g.n_out;
  a.sys_list = nullptr;
  a.n_list = 1;
  a.t_first = g.t_first;
  const int64_t nseq_total = (int64_t)(g.n_sys_total > 0 ? g.n_sys_total : 1) * g.batch;
  for (int s = 0; s < g.n_src; ++s) {
    a.K[s] = g.src[s].K;
    a.shift[s] = g.src[s].shift;
    a.w_plane_off[s] = g.src[s].w_plane_off;
    a.w_plane_stride[s] = 0;
    a.a_row0[s] = (int)g.src[s].row0;
    if (!map3d(&maps.A[s], g.src[s].A, true, g.src[s].K, g.src[s].row0 + g.L, nseq_total, HM)) return CASC_ERR_CUDA;
    const int64_t planes = g.src[s].w_planes > 0 ? g.src[s].w_planes : 2;
    if (!map3d(&maps.W[s], g.src[s].W, true, g.src[s].K, g.n_out, planes, BN / 2)) return CASC_ERR_CUDA;
  }
  a.has_residual = g.R != nullptr;
  a.peer_out = g.peer_out; a.peer_l_begin = g.peer_l_begin; a.peer_shift = g.peer_shift;
  a.r_row0 = (int)g.R_row0;
  a.out_row0 = (int)g.out_row0;
  if (g.R && !map3d(&maps.R, g.R, true, g.n_out, g.R_row0 + g.L, nseq_total, HM)) return CASC_ERR_CUDA;
  if (!map3d(&maps.out, g.out, true, g.n_out, g.out_row0 + g.L, nseq_total, HM)) return CASC_ERR_CUDA;
  if (cudaFuncSetAttribute(mimo_gemm_pair_tf32_kernel<BN, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)C::SMEM) != cudaSuccess)
    return CASC_ERR_CUDA;
  const int64_t blocks = (g.L + 2 * HM - 1) / (2 * HM) - g.t_first / 2;
  const int64_t tiles = (int64_t)g.batch * blocks * (g.n_out / BN);
  if (tiles <= 0) return CASC_OK;
  const int pairs = (int)std::min<int64_t>(tiles, 74);
  mimo_gemm_pair_tf32_kernel<BN, SPLIT><<<2 * pairs, THREADS, C::SMEM, st>>>(maps, a);
  CASC_LAUNCHED();
  return CASC_OK;
}

int launch_mimo_gemm_pair_tf32(const MimoGemm& g, cudaStream_t st) {
  int K = 0;
  for (int s = 0; s < g.n_src; ++s) K += g.src[s].K;
  // contractions longer than 512 (E3: 256) split the main chain (PCfg) to keep fp32 accuracy
  return K > 512 ? launch_pt<128, 3>(g, st) : launch_pt<128, 1>(g, st);
}

}  // namespace casc
