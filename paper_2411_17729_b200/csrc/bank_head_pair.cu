// Bank head (stages 0..Kc-1 with Bbar u, R22) on CTA PAIRS (m = 64):
//
//   v^(Kc)_l = sum_{j < 128} (Abar^j Bbar) u_{l-j}     (the expanded product of PAPER.md:126)
//
// The same per-tile K = 128 Toeplitz GEMM as bank_head_ws.cu (3xTF32, the Toeplitz operand Z a
// 4 KB shared-memory buffer read with LBO = 64 B), but two consecutive 128-step tiles form one
// M = 256 MMA (tcgen05.mma.cta_group::2) over a cluster of two CTAs. The Krylov operand (B) is
// split between the pair: for hi.[hi | lo] (N = 128) the leader holds the 64 hi rows and the peer
// the 64 lo rows; for lo.hi (N = 64) each holds 32 of the hi rows. Each SM then reads 11 KB of MMA
// operands per K step instead of 14 KB -- shared-memory bandwidth bounds the one-CTA head.
// Roles per CTA (192 threads, two CTAs per SM):
//   warp 0     builds Z for its tile of the next pairs into a 2-slot ring (u staged in smem) and
//              arrives on the leader's z_full
//   warp 1     (leader) issues the 32 MMAs of a tile pair; commits are multicast to both CTAs
//   warps 2-5  drain TMEM into a SWIZZLE_128B staging tile and TMA-store it (or write the output
//              parts, R24-R26); they release the accumulator on the leader's tempty
#include <cuda.h>

#include "common.cuh"
#include "sm100.cuh"
#include "bank_tc.cuh"
#include "mimo_tc.cuh"

namespace casc {
using namespace sm100;

namespace {
constexpr int TM = 128, KL = 128, ZR = 256, MS = 64, BCH = KL / 4;
__device__ __forceinline__ void named_sync_p(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void tma_store_3d_p(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];"
               ::"l"(map), "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ uint32_t cta_rank_p() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_p() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {        // both CTAs' barrier at this offset
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
__device__ __forceinline__ void arrive_on_leader(uint64_t* bar, bool is_leader) {
  if (is_leader) {
    mbar_arrive(bar);
    return;
  }
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");   // CTA scope
}
}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 2)
    bank_head_pair_kernel(const __grid_constant__ CUtensorMap vmap, BankHeadArg a, int pairs_per_cluster) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* Stg = reinterpret_cast<float*>(smem);                 // [128 rows][32] SW128 half tile, 16 KB
  float* Bp = Stg + TM * 32;                                   // [BCH][64 rows][4]: hi (leader) | lo (peer)
  float* Bq = Bp + BCH * 64 * 4;                               // [BCH][32 rows][4]: hi rows 32*rank ..
  float* Zb = Bq + BCH * 32 * 4;                               // [2 slots][hi|lo][ZR][4]
  float* Us = Zb + 2 * 2 * ZR * 4;                             // [2 slots][264] u window
  __shared__ uint64_t z_full[2], z_empty[2], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid / 32, 0), lane = tid % 32;
  const uint32_t rank = cta_rank_p();
  const bool is_leader = rank == 0;
  const int li = blockIdx.y / a.batch, b = blockIdx.y % a.batch;
  const int c = a.sys_list[li];
  const int seq = c * a.batch + b;
  const float* u = a.u + (int64_t)seq * a.L;

  {                                                            // this CTA's part of the Krylov operand
    const float* kh = a.krT + (int64_t)c * 2 * MS * KL;
    const float* kp = kh + (is_leader ? 0 : MS * KL);          // hi | lo
    for (int e = tid; e < 64 * BCH; e += 192) {
      const int ch = e / 64, n = e % 64;
      *reinterpret_cast<float4*>(Bp + (ch * 64 + n) * 4) = __ldg(reinterpret_cast<const float4*>(kp + n * KL + ch * 4));
    }
    for (int e = tid; e < 32 * BCH; e += 192) {
      const int ch = e / 32, n = e % 32;
      *reinterpret_cast<float4*>(Bq + (ch * 32 + n) * 4) =
          __ldg(reinterpret_cast<const float4*>(kh + (32 * rank + n) * KL + ch * 4));
    }
  }
  fence_async_smem();
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&z_full[s], 2 * 32);
      mbar_init(&z_empty[s], 1);
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(4 * MS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_p();                                            // both CTAs' barriers, operands and TMEM ready
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {                                              // the pair's MMAs address both TMEMs alike
    uint32_t peer_addr, peer_base;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer_addr) : "r"(smem_u32(&tmem_base)), "r"(rank ^ 1u));
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(peer_base) : "r"(peer_addr) : "memory");
    if (peer_base != tbase) __trap();
  }

  const int64_t ntiles = (a.L + TM - 1) / TM;
  const int64_t npairs = (ntiles + 1) / 2;
  const int64_t pair_begin = (int64_t)(blockIdx.x / 2) * pairs_per_cluster;
  const int64_t pair_end = npairs < pair_begin + pairs_per_cluster ? npairs : pair_begin + pairs_per_cluster;
  const int nt = (int)(pair_end - pair_begin);
  auto tile_of = [&](int i) -> int64_t { return 2 * (pair_begin + i) + rank; };   // may be >= ntiles (zeros)

  if (warp == 0) {
    // ---------------------------------------------------------------- Z producer (both CTAs)
    float ur[9];
    auto load_u = [&](int i) {                    // u[t0-127 .. t0+160] (259 used)
      const int64_t base = tile_of(i) * TM - (KL - 1);
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const int64_t t = base + lane + 32 * q;
        ur[q] = (i < nt && t >= 0 && t < a.L) ? __ldg(u + t) : 0.f;
      }
    };
    load_u(0);
    for (int i = 0; i < nt; ++i) {
      const int slot = i & 1;
      if (i >= 2) mbar_wait(&z_empty[slot], (uint32_t)(((i - 2) >> 1) & 1));
      float* us = Us + slot * 264;
#pragma unroll
      for (int q = 0; q < 9; ++q)
        if (lane + 32 * q < 264) us[lane + 32 * q] = ur[q];
      __syncwarp();
      load_u(i + 1);                              // prefetch the next window
      float* zh = Zb + slot * 2 * ZR * 4;
      float* zl = zh + ZR * 4;
#pragma unroll
      for (int r = 0; r < 8; ++r) {               // Z-row w = (u[t0-127+w+q], q = 0..3)
        const int w = lane + 32 * r;
        const float4 z = make_float4(us[w], us[w + 1], us[w + 2], us[w + 3]);
        const float4 h = tf32_hi4(z);
        *reinterpret_cast<float4*>(zh + w * 4) = h;
        *reinterpret_cast<float4*>(zl + w * 4) = tf32_lo4(z, h);
      }
      fence_async_smem();
      arrive_on_leader(&z_full[slot], is_leader);
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader, whole warp)
    if (is_leader) {
      const uint32_t idesc = make_idesc(FMT_TF32, 2 * TM, MS), idesc2 = make_idesc(FMT_TF32, 2 * TM, 2 * MS);
      const uint32_t bp = smem_u32(Bp), bq = smem_u32(Bq);
      for (int i = 0; i < nt; ++i) {
        const int slot = i & 1;
        mbar_wait_u(&z_full[slot], (uint32_t)((i >> 1) & 1));
        mbar_wait_u(&tempty[slot], (uint32_t)(((i >> 1) & 1) ^ 1));
        tc_fence_after();
        const uint32_t zh = smem_u32(Zb + slot * 2 * ZR * 4), zl = zh + ZR * 16;
        const uint32_t acc = tbase + slot * 2 * MS;
#pragma unroll 4
        for (int ks = 0; ks < KL / 8; ++ks) {
          const uint64_t azh = make_sdesc(zh + ks * 128, 64, 128, LAYOUT_NONE);
          const uint64_t azl = make_sdesc(zl + ks * 128, 64, 128, LAYOUT_NONE);
          const uint64_t bpd = make_sdesc(bp + ks * 2 * 64 * 16, 64 * 16, 128, LAYOUT_NONE);
          const uint64_t bqd = make_sdesc(bq + ks * 2 * 32 * 16, 32 * 16, 128, LAYOUT_NONE);
          mma_tf32_pair(acc, azh, bpd, idesc2, ks > 0);          // [hi.hi | hi.lo]
          mma_tf32_pair(acc + MS, azl, bqd, idesc, 1);          // corr += lo.hi
        }
        commit_pair(&z_empty[slot]);
        commit_pair(&tfull[slot]);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..5, both CTAs)
    const int q = warp & 3, row = q * 32 + lane;
    const bool leader_t = (warp == 2 && lane == 0);
    int depth = 0;
    bool to_parts = false;
    if (a.op.planes != nullptr) {
      const int ne = a.op.neff[c], kc = a.op.kc[c];
      depth = fold_depth(ne, kc, a.op.fold);
      to_parts = ne - depth == kc;
    }
    for (int i = 0; i < nt; ++i) {
      const int slot = i & 1;
      mbar_wait_u(&tfull[slot], (uint32_t)((i >> 1) & 1));
      tc_fence_after();
      float v[MS], vc[MS];
      const uint32_t tacc = tbase + ((uint32_t)(q * 32) << 16) + slot * 2 * MS;
#pragma unroll
      for (int c0 = 0; c0 < MS; c0 += 16) tmem_ld16(tacc + c0, v + c0);
#pragma unroll
      for (int c0 = 0; c0 < MS; c0 += 16) tmem_ld16(tacc + MS + c0, vc + c0);
#pragma unroll
      for (int n = 0; n < MS; ++n) v[n] += vc[n];             // main + corr (round to nearest)
      tc_fence_before();
      arrive_on_leader(&tempty[slot], is_leader);
      const int64_t tile = tile_of(i);
      if (to_parts) {                             // the 2^(depth+1) output parts instead of v
        const int64_t l = tile * TM + row;
        const float* vb = a.op.vec + (int64_t)c * kMaxParts * MS;
        const int np = 2 << depth;
        for (int bp = 0; bp < np; ++bp) {
          float p = 0.f;
#pragma unroll
          for (int n = 0; n < MS; n += 4) {
            const float4 c4 = __ldg(reinterpret_cast<const float4*>(vb + bp * MS + n));
            p = fmaf(c4.x, v[n], p); p = fmaf(c4.y, v[n + 1], p); p = fmaf(c4.z, v[n + 2], p); p = fmaf(c4.w, v[n + 3], p);
          }
          if (l < a.L) a.op.planes[bp * a.op.plane + (int64_t)seq * a.L + l] = p;
        }
        continue;
      }
      if (tile >= ntiles) continue;               // the pair's second tile past the sequence end
#pragma unroll
      for (int h = 0; h < 2; ++h) {               // two SW128 halves of 32 fp32 columns
        if (leader_t) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        named_sync_p(1, 128);
        uint8_t* rrow = reinterpret_cast<uint8_t*>(Stg) + row * 128;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          *reinterpret_cast<float4*>(rrow + ((cc ^ (row & 7)) * 16)) =
              make_float4(v[32 * h + 4 * cc], v[32 * h + 4 * cc + 1], v[32 * h + 4 * cc + 2], v[32 * h + 4 * cc + 3]);
        fence_async_smem();
        named_sync_p(1, 128);
        if (leader_t) {
          tma_store_3d_p(&vmap, Stg, 32 * h, (int)(tile * TM), seq);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (leader_t) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_p();                                            // no CTA of the pair still uses TMEM
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(4 * MS) : "memory");
}

int launch_bank_head_pair(int m, const BankHeadArg& a, int64_t n_seq_total, cudaStream_t st) {
  if (m != 64) return CASC_ERR_UNSUPPORTED;
  if (a.n_list <= 0) return CASC_OK;
  if (a.n_list * (int64_t)a.batch > 65535) return CASC_ERR_UNSUPPORTED;
  CUtensorMap vmap;
  if (!map3d(&vmap, a.V, true, 64, a.L, n_seq_total, TM)) return CASC_ERR_CUDA;
  const size_t smem = 1024 + (size_t)(TM * 32 + BCH * 64 * 4 + BCH * 32 * 4 + 2 * 2 * ZR * 4 + 2 * 264) * sizeof(float);
  if (cudaFuncSetAttribute(bank_head_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return CASC_ERR_CUDA;
  const int64_t npairs = ceil_div(ceil_div(a.L, TM), 2);
  const int ppc = a.tiles_per_cta > 1 ? a.tiles_per_cta / 2 : 1;
  dim3 grid((unsigned)(2 * ceil_div(npairs, ppc)), (unsigned)(a.n_list * a.batch));
  bank_head_pair_kernel<<<grid, 192, smem, st>>>(vmap, a, ppc);
  CASC_LAUNCHED();
  return CASC_OK;
}

}  // namespace casc
