// Shifted multi-source GEMM, bf16, on CTA PAIRS (tcgen05 cta_group::2): the large-m MIMO steps
// (E4: m = 1024) of PAPER.md:185-229, the same map as mimo_tc.cu
//   out[s][l][n] = sum_src sum_k A_src[s][l - shift_src][k] W_src[n][k]  (+ R[s][l][n])
// with 256 x 256 output tiles computed by a cluster of two CTAs: each CTA stages 128 rows of A
// and 128 rows (output columns) of W per 64-wide K chunk, and the leader CTA issues one
// M = 256, N = 256, K = 16 MMA that reads both CTAs' shared memory and accumulates each CTA's
// 128 rows in its own TMEM. Against the one-CTA kernel (128 x 256 tiles) every CTA moves half the
// W bytes per K chunk, so a 32 KB ring slot replaces a 48 KB one: five slots cover 2.5k MMA
// cycles instead of three covering 1.5k (the one-CTA kernel's MMA warp waited on operands ~58% of
// the time, CASC_GEMM_DBG), and L2 -> SM traffic per flop drops by a third.
//
// Protocol (as CUTLASS's 2-SM kernels): both CTAs' TMA loads signal the LEADER's full barrier
// (its shared::cluster address from mapa); the leader's producer posts the
// expected bytes of both halves; MMA completion is multicast to both CTAs' empty barriers and,
// per tile, to both CTAs' accumulator-full barriers; both CTAs' epilogue threads arrive on the
// leader's accumulator-empty barrier (remote arrive through mapa). Residual/staging rings are
// per CTA. TMEM (2 x 256 columns) is allocated by both CTAs with cta_group::2.
#include <cuda.h>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"
#include "mimo_tc.cuh"

namespace casc {
using namespace sm100;

namespace {
constexpr int HM = 128;                  // rows per CTA
constexpr int BN = 256;                  // output columns per pair tile
constexpr int BK = 64;                   // bf16 K per chunk (128-byte rows)
constexpr uint32_t A_BYTES = HM * 128;   // 16 KB
constexpr uint32_t W_BYTES = 128 * 128;  // 16 KB: this CTA's 128 output columns
constexpr uint32_t STAGE_BYTES = A_BYTES + W_BYTES;
constexpr int RS = 4;                    // residual / staging chunks (16 KB)
constexpr uint32_t R_BYTES = HM * 128;
constexpr int STAGES = (int)((226u * 1024u - 1024u - RS * R_BYTES) / STAGE_BYTES) < 8
                           ? (int)((226u * 1024u - 1024u - RS * R_BYTES) / STAGE_BYTES) : 8;
constexpr int CW = 64;                   // epilogue chunk width (bf16 columns = 128 bytes)
constexpr int NCH = BN / CW;
constexpr int R_WARP = 6;
constexpr int THREADS = 32 * (R_WARP + 1);
constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + RS * R_BYTES;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2sm(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_load_1(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];"
               ::"l"(map), "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void bulk_commit2() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read2() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait2() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void named_sync2(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void mma_f16_pair_w(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// arrive on the barrier at this offset in both CTAs of the pair once the issued MMAs complete
__device__ __forceinline__ void mma_commit_pair_w(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {   // arrive on the leader CTA's copy
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  // default semantics (release, CTA scope): a cluster-scope release compiles to MEMBAR.ALL.GPU
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void tmem_ld32_2(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ uint32_t pack_bf16_2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_bf16_2(uint32_t u) {
  __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&u);
  return __bfloat1622float2(h);
}

struct PairCoord {
  int seq, l0, nb;     // l0: first row of this CTA's half
};
__device__ __forceinline__ PairCoord decode2(int64_t tile, const MimoArg& a, int n_nblk, int64_t nb_eff, int t0_blk,
                                             uint32_t rank) {
  PairCoord t;
  t.nb = (int)(tile % n_nblk);
  const int64_t r = tile / n_nblk;
  t.l0 = (int)((t0_blk + r % nb_eff) * (2 * HM) + rank * HM);
  const int64_t sidx = r / nb_eff;
  const int li = (int)(sidx / a.batch), b = (int)(sidx % a.batch);
  const int sys = a.sys_list ? a.sys_list[li] : 0;
  t.seq = sys * a.batch + b;
  return t;
}
}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    mimo_gemm_pair_kernel(const __grid_constant__ MimoMaps maps, MimoArg a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sR = smem + STAGES * STAGE_BYTES;
  __shared__ uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2], rfull[RS], rempty[RS];
  __shared__ uint32_t tmem_base;
  auto stA = [&](int s) { return smem + s * STAGE_BYTES; };
  auto stW = [&](int s) { return smem + s * STAGE_BYTES + A_BYTES; };

  // warp index broadcast from lane 0: provably warp-uniform, so role branches are uniform control
  // flow and ptxas keeps role-local uniform values (descriptors, TMEM addresses) in uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const uint32_t rank = cta_rank();
  const bool is_leader = rank == 0;
  const int64_t blocks_per_b = (a.L + 2 * HM - 1) / (2 * HM);
  const int t0_blk = a.t_first / 2;                       // 256-row blocks (an extra 128 rows may be recomputed)
  const int64_t nb_eff = blocks_per_b - t0_blk;
  const int n_nblk = (a.n_out + BN - 1) / BN;
  const int64_t n_tiles = (int64_t)a.n_list * a.batch * nb_eff * n_nblk;
  const int64_t pair = blockIdx.x / 2, n_pairs = gridDim.x / 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 2 * 128); }
    for (int s = 0; s < RS; ++s) { mbar_init(&rfull[s], 1); mbar_init(&rempty[s], 1); }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();                                          // both CTAs' barriers and TMEM ready
  tc_fence_after();
  if (tmem_base != 0) __trap();                            // 512 columns: the whole TMEM
  constexpr uint32_t tbase = 0;

  if (warp == 0) {
    // =========================================================== TMA producer (both CTAs)
    {                                         // whole warp loops, lane 0 issues (uniform MMA operands, mimo_tc.cu)
      const bool issue = lane == 0;
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = pair; t < n_tiles; t += n_pairs) {
        const PairCoord tc = decode2(pair_tile_order(t, n_pairs, n_nblk, n_tiles), a, n_nblk, nb_eff, t0_blk, rank);
        for (int src = 0; src < a.n_src; ++src) {
          const int nk = a.K[src] / BK;
          const int plane = a.w_plane_off[src];
          for (int kc = 0; kc < nk; ++kc) {
            mbar_wait(&empty[s], ph ^ 1);
            if (issue) {
              if (is_leader) mbar_arrive_expect_tx(&full[s], 2 * STAGE_BYTES);
              uint32_t fb;                          // the leader CTA's full[s] (shared::cluster)
              asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(fb) : "r"(smem_u32(&full[s])));
              tma_load_2sm(stA(s), &maps.A[src], fb, kc * BK, a.a_row0[src] + tc.l0 - (int)a.shift[src], tc.seq);
              tma_load_2sm(stW(s), &maps.W[src], fb, kc * BK, tc.nb * BN + (int)rank * 128, plane);
            }
            if (++s == STAGES) { s = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == R_WARP) {
    // =========================================================== residual / staging producer (per CTA)
    {
      const bool issue = lane == 0;
      int rs = 0;
      uint32_t rph = 0;
      for (int64_t t = pair; t < n_tiles; t += n_pairs) {
        const PairCoord tc = decode2(pair_tile_order(t, n_pairs, n_nblk, n_tiles), a, n_nblk, nb_eff, t0_blk, rank);
        for (int j = 0; j < NCH; ++j) {
          mbar_wait(&rempty[rs], rph ^ 1);
          if (!issue) {
          } else if (a.has_residual) {
            mbar_arrive_expect_tx(&rfull[rs], R_BYTES);
            tma_load_1(sR + rs * R_BYTES, &maps.R, &rfull[rs], tc.nb * BN + j * CW, a.r_row0 + tc.l0, tc.seq);
          } else {
            mbar_arrive(&rfull[rs]);
          }
          if (++rs == RS) { rs = 0; rph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // =========================================================== MMA issuer (leader CTA, whole warp)
    if (is_leader) {
      const uint32_t idesc = make_idesc(FMT_BF16, 2 * HM, BN);
      int s = 0;
      uint32_t ph = 0;
      int64_t t_local = 0;
      for (int64_t t = pair; t < n_tiles; t += n_pairs, ++t_local) {
        const int acc = (int)(t_local & 1);
        mbar_wait(&tempty[acc], (uint32_t)((t_local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tbase + acc * BN;
        bool first = true;
        for (int src = 0; src < a.n_src; ++src) {
          const int nk = a.K[src] / BK;
          for (int kc = 0; kc < nk; ++kc) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint64_t ad0 = make_sdesc(smem_u32(stA(s)), 16, 1024, LAYOUT_SW128);
            const uint64_t wd0 = make_sdesc(smem_u32(stW(s)), 16, 1024, LAYOUT_SW128);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              mma_f16_pair_w(d, sdesc_add(ad0, k * 32), sdesc_add(wd0, k * 32), idesc, first ? 0u : 1u);
              first = false;
            }
            mma_commit_pair_w(&empty[s]);
            if (++s == STAGES) { s = 0; ph ^= 1; }
          }
        }
        mma_commit_pair_w(&tfull[acc]);
      }
    }
  } else if (warp >= 2 && warp <= 5) {
    // =========================================================== epilogue (warps 2..5, both CTAs)
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const bool leader_t = (warp == 2 && lane == 0);
    int64_t t_local = 0;
    int rs = 0, prev_rs = -1;
    uint32_t rph = 0;
    for (int64_t t = pair; t < n_tiles; t += n_pairs, ++t_local) {
      const PairCoord tc = decode2(pair_tile_order(t, n_pairs, n_nblk, n_tiles), a, n_nblk, nb_eff, t0_blk, rank);
      const int acc = (int)(t_local & 1);
      mbar_wait(&tfull[acc], (uint32_t)((t_local >> 1) & 1));
      tc_fence_after();
      for (int j = 0; j < NCH; ++j) {
        uint8_t* rbuf = sR + rs * R_BYTES;
        uint32_t v[64];
        const uint32_t taddr = tbase + ((uint32_t)(q * 32) << 16) + acc * BN + j * CW;
        tmem_ld32_2(taddr, v);
        tmem_ld32_2(taddr + 32, v + 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (j == NCH - 1) {                       // accumulator drained: release it to the leader's MMA
          tc_fence_before();
          if (is_leader) mbar_arrive(&tempty[acc]);
          else mbar_arrive_leader(&tempty[acc]);
        }
        mbar_wait(&rfull[rs], rph);
        uint8_t* rrow = rbuf + row * 128;
        // this row also goes to the successor rank's halo rows (peer halo, seqshard.cu): straight
        // from registers over the peer mapping (NVLink), as the tile is produced
        const int64_t lrow = (int64_t)tc.l0 + row;
        __nv_bfloat16* prow = (a.peer_out && lrow >= a.peer_l_begin && lrow < a.L)
            ? static_cast<__nv_bfloat16*>(a.peer_out) + ((int64_t)tc.seq * (a.out_row0 + a.L) + a.out_row0 + lrow - a.peer_shift) * a.n_out + tc.nb * BN + j * CW
            : nullptr;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint4* p = reinterpret_cast<uint4*>(rrow + ((c ^ (row & 7)) * 16));
          float f[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(v[c * 8 + e]);
          if (a.has_residual) {
            const uint4 r = *p;
            const float2 r0 = unpack_bf16_2(r.x), r1 = unpack_bf16_2(r.y), r2 = unpack_bf16_2(r.z), r3 = unpack_bf16_2(r.w);
            f[0] += r0.x; f[1] += r0.y; f[2] += r1.x; f[3] += r1.y;
            f[4] += r2.x; f[5] += r2.y; f[6] += r3.x; f[7] += r3.y;
          }
          *p = make_uint4(pack_bf16_2(f[0], f[1]), pack_bf16_2(f[2], f[3]), pack_bf16_2(f[4], f[5]), pack_bf16_2(f[6], f[7]));
          if (prow) *reinterpret_cast<uint4*>(prow + 8 * c) = *p;
        }
        fence_async_smem();
        named_sync2(1, 128);
        if (leader_t) {
          tma_store(&maps.out, rbuf, tc.nb * BN + j * CW, a.out_row0 + tc.l0, tc.seq);
          bulk_commit2();
          if (prev_rs >= 0) {
            bulk_wait_read2<1>();
            mbar_arrive(&rempty[prev_rs]);
          }
        }
        prev_rs = rs;
        if (++rs == RS) { rs = 0; rph ^= 1; }
      }
    }
    if (leader_t) bulk_wait2<0>();
    if (a.peer_out) __threadfence_system();       // peer stores visible before the kernel completes
  }
  tc_fence_before();
  cluster_sync();                                          // no CTA of the pair still uses TMEM
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512) : "memory");
}

bool mimo_pair_ok(const MimoGemm& g, bool tf32) {
  if (tf32 || g.n_out % 256 != 0 || g.w_resident || g.ab) return false;
  for (int s = 0; s < g.n_src; ++s)
    if (g.src[s].K % BK || g.src[s].w_plane_stride != 0) return false;   // one weight plane per source
  return g.sys_list == nullptr;
}

int launch_mimo_gemm_pair(const MimoGemm& g, cudaStream_t st) {
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
  const int64_t nseq_total = g.batch;
  for (int s = 0; s < g.n_src; ++s) {
    a.K[s] = g.src[s].K;
    a.shift[s] = g.src[s].shift;
    a.w_plane_off[s] = g.src[s].w_plane_off;
    a.w_plane_stride[s] = 0;
    a.a_row0[s] = (int)g.src[s].row0;
    if (!map3d(&maps.A[s], g.src[s].A, false, g.src[s].K, g.src[s].row0 + g.L, nseq_total, HM)) return CASC_ERR_CUDA;
    const int64_t planes = g.src[s].w_planes > 0 ? g.src[s].w_planes : 1;
    if (!map3d(&maps.W[s], g.src[s].W, false, g.src[s].K, g.n_out, planes, 128)) return CASC_ERR_CUDA;
  }
  a.has_residual = g.R != nullptr;
  a.r_row0 = (int)g.R_row0;
  a.out_row0 = (int)g.out_row0;
  a.peer_out = g.peer_out; a.peer_l_begin = g.peer_l_begin; a.peer_shift = g.peer_shift;
  if (g.R && !map3d(&maps.R, g.R, false, g.n_out, g.R_row0 + g.L, nseq_total, HM)) return CASC_ERR_CUDA;
  if (!map3d(&maps.out, g.out, false, g.n_out, g.out_row0 + g.L, nseq_total, HM)) return CASC_ERR_CUDA;
  if (cudaFuncSetAttribute(mimo_gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) != cudaSuccess)
    return CASC_ERR_CUDA;
  const int64_t blocks = (g.L + 2 * HM - 1) / (2 * HM) - g.t_first / 2;
  const int64_t tiles = (int64_t)g.batch * blocks * (g.n_out / BN);
  if (tiles <= 0) return CASC_OK;
  const int pairs = (int)std::min<int64_t>(tiles, 74);
  mimo_gemm_pair_kernel<<<2 * pairs, THREADS, SMEM, st>>>(maps, a);
  CASC_LAUNCHED();
  return CASC_OK;
}

}  // namespace casc
