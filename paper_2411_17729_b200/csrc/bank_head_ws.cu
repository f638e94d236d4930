// Bank head (stages 0..Kc-1 with Bbar u, R22), warp-specialized (m = 64):
//
//   v^(Kc)_l = sum_{j < 128} (Abar^j Bbar) u_{l-j}     (the expanded product of PAPER.md:126)
//
// per 128-step tile one K = 128 GEMM on the fp16 tensor path (kind::f16, fp32 accumulate) with the
// operands split in two fp16 parts, x = hi + lo (hi = rn(x), lo = rn(x - hi): 22 significant bits,
// as the 3xTF32 split; R33): hi.hi + lo.hi + hi.lo at twice the tf32 MMA rate. fp16's
// range is handled by exact power-of-two scales: the Krylov weights per state column n
// (max_j |W_jn| scaled into [2^14, 2^15)), the Toeplitz tile per tile (its u window likewise); the
// epilogue multiplies the fp32 accumulators back by the inverse powers of two. The A operand, the
// Toeplitz matrix u_{l-j}, is a 4 KB shared-memory buffer Z (16-B rows of 8 fp16) read with
// LBO = 128 B (row r, K chunk c' = Z-row r + 8c'). The weights are stored hi and lo stacked along
// N ([K chunk][hi 64 | lo 64 rows]), so Z_hi x [B_hi | B_lo] is one N = 128 MMA writing hi.hi to the
// main and hi.lo to the correction accumulator, and Z_lo x B_hi (N = 64) adds to the correction.
// Roles (192 threads, two CTAs per SM):
//   warp 0     builds Z (and the tile's scale) for the next tiles into a 2-slot ring (u staged
//              through shared memory)
//   warp 1     issues the 16 MMAs of a tile into one of two TMEM accumulators (main | corr)
//   warps 2-5  drain TMEM (lane = time row) into a SWIZZLE_128B staging tile and TMA-store it
// Each CTA walks `tiles_per_cta` consecutive tiles of one sequence, so the Krylov weights
// (32 KB of fp16 hi/lo, split from the float64 weights in the prologue) are built once per CTA.
#include <cuda.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "sm100.cuh"
#include "bank_tc.cuh"
#include "mimo_tc.cuh"

namespace casc {
using namespace sm100;

namespace {
constexpr int TM = 128, KL = 128, ZR = 256;
__device__ __forceinline__ void named_sync_h(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void tma_store_3d_h(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];"
               ::"l"(map), "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void bulk_commit_h() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
}  // namespace

template <int MS>
__global__ void __launch_bounds__(192, 2) bank_head_ws_kernel(const __grid_constant__ CUtensorMap vmap, BankHeadArg a) {
  static_assert(MS == 64, "TMA-store epilogue written for m = 64");
  constexpr int BCH = KL / 8;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps the shared state space (STS/LDS, not generic ST/LD)
  float* Stg = reinterpret_cast<float*>(smem);                 // [128 rows][32] SW128 half tile, 16 KB
  __half* Bc = reinterpret_cast<__half*>(Stg + TM * 32);       // [BCH][hi MS | lo MS][8] fp16, 32 KB
  __half* Zb = Bc + 2 * KL * MS;                               // [2 slots][hi|lo][ZR][8] fp16
  float* Us = reinterpret_cast<float*>(Zb + 2 * 2 * ZR * 8);   // [2 slots][264] u window
  __shared__ uint64_t z_full[2], z_empty[2], tfull[2], tempty[2], sc_full[4], w_full;
  __shared__ uint32_t tmem_base;
  __shared__ float col_inv[MS], tile_inv[4];                   // inverse scales (powers of two)

  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid / 32, 0), lane = tid % 32;
  const int li = blockIdx.y / a.batch, b = blockIdx.y % a.batch;
  const int c = a.sys_list[li];
  const int seq = c * a.batch + b;
  const float* u = a.u + (int64_t)seq * a.L;

  // the channel's fp16 Krylov weights (bank_derived_kernel): 32 KB by one bulk copy
  const __half* kw = a.kr16 + (int64_t)c * 2 * KL * MS;
  if (tid == 0) {
    mbar_init(&w_full, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&w_full, 2 * KL * MS * 2);
    bulk_g2s(Bc, kw, 2 * KL * MS * 2, &w_full);
  }
  if (tid < MS) col_inv[tid] = __ldg(a.kinv + (int64_t)c * MS + tid);
  fence_async_smem();
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&z_full[s], 32);
      mbar_init(&z_empty[s], 1);
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
    }
    for (int s = 0; s < 4; ++s) mbar_init(&sc_full[s], 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<4 * MS>(&tmem_base);         // 2 slots x (main | corr)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  const int64_t ntiles = (a.L + TM - 1) / TM;
  const int64_t tile_begin = (int64_t)blockIdx.x * a.tiles_per_cta;
  const int64_t tile_end = ntiles < tile_begin + a.tiles_per_cta ? ntiles : tile_begin + a.tiles_per_cta;
  const int nt = (int)(tile_end - tile_begin);

  if (warp == 0) {
    // ---------------------------------------------------------------- Z producer
    // Window of tile i: W_i[w] = u[t0_i - 127 + w], w < 259 (Z-row w reads W_i[w .. w + 3]). The next
    // window is this one shifted by 128: W_{i+1}[w] = W_i[w + 128] for w < 131, and 128 new values
    // W_{i+1}[131 .. 259) = u[t0_i + 132 ..) -- so after the CTA's first tile each tile reads 128
    // values of u, not 259.
    float nr[4];
    auto load_new = [&](int i) {                  // W_i[131 .. 259)
      const int64_t base = (tile_begin + i) * TM - (KL - 1) + 131;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t t = base + lane + 32 * q;
        nr[q] = (i < nt && t >= 0 && t < a.L) ? __ldg(u + t) : 0.f;
      }
    };
    {                                             // the first window in full
      const int64_t base = tile_begin * TM - (KL - 1);
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const int64_t t = base + lane + 32 * q;
        if (lane + 32 * q < 264) Us[lane + 32 * q] = (nt > 0 && t >= 0 && t < a.L) ? __ldg(u + t) : 0.f;
      }
      load_new(1);
      __syncwarp();
    }
    for (int i = 0; i < nt; ++i) {
      const int slot = i & 1;
      if (i >= 2) mbar_wait(&z_empty[slot], (uint32_t)(((i - 2) >> 1) & 1));
      float* us = Us + slot * 264;
      __half* zh = Zb + slot * 2 * ZR * 8;
      __half* zl = zh + ZR * 8;
      // the tile's scale: max |u| over the window the MMAs read (Z-rows 0..247 -> W_i[0 .. 255))
      uint32_t mb = 0;
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (lane + 32 * r < 255) mb = max(mb, __float_as_uint(fabsf(us[lane + 32 * r])));
      mb = __reduce_max_sync(0xffffffffu, mb);
      const float mx = __uint_as_float(mb);
      // (exponents clamped to +-110 so that the scale and its inverse stay normal fp32 numbers: a
      // window below 2^-110 in magnitude keeps only fp16's subnormal precision; inf / NaN propagate)
      const int et = mx > 0.f ? max(-110, min(110, ilogbf(mx))) : 0;
      const float sc = ldexpf(1.f, 14 - et);
      // 4-deep ring: this write (tile i) follows z_empty of tile i - 2 (the MMA warp's commit), whose
      // MMAs waited for tempty of tile i - 4, which the epilogue arrives after reading tile_inv[i & 3]
      if (lane == 0) tile_inv[i & 3] = ldexpf(1.f, et - 14);
#pragma unroll
      for (int r = 0; r < 8; ++r) {               // Z-row w = (u[t0-127+w+q] * 2^(14 - et), q = 0..7)
        const int w = lane + 32 * r;
        __align__(16) __half2 h[4], l[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float x0 = us[w + 2 * q] * sc, x1 = us[w + 2 * q + 1] * sc;
          h[q] = __floats2half2_rn(x0, x1);
          const float2 hf = __half22float2(h[q]);
          l[q] = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
        }
        *reinterpret_cast<uint4*>(zh + w * 8) = *reinterpret_cast<const uint4*>(h);
        *reinterpret_cast<uint4*>(zl + w * 8) = *reinterpret_cast<const uint4*>(l);
      }
      fence_async_smem();
      mbar_arrive(&z_full[slot]);
      if (lane == 0) mbar_arrive(&sc_full[i & 3]);   // the epilogue's inverse scale of tile i
      if (i + 1 < nt) {                           // W_{i+1} into the other slot
        float* un = Us + (slot ^ 1) * 264;
#pragma unroll
        for (int q = 0; q < 5; ++q)
          if (lane + 32 * q < 131) un[lane + 32 * q] = us[lane + 32 * q + 128];
#pragma unroll
        for (int q = 0; q < 4; ++q) un[131 + lane + 32 * q] = nr[q];
        load_new(i + 2);                          // prefetch the next new values
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    {                                             // whole warp: operands stay in uniform registers
      const uint32_t idesc = make_idesc(FMT_F16, TM, MS), idesc2 = make_idesc(FMT_F16, TM, 2 * MS);
      const uint32_t bc = smem_u32(Bc);
      mbar_wait_u(&w_full, 0);                     // weights landed (async proxy: visible to the MMAs)
      for (int i = 0; i < nt; ++i) {
        const int slot = i & 1;
        mbar_wait_u(&z_full[slot], (uint32_t)((i >> 1) & 1));
        mbar_wait_u(&tempty[slot], (uint32_t)(((i >> 1) & 1) ^ 1));
        tc_fence_after();
        const uint32_t zh = smem_u32(Zb + slot * 2 * ZR * 8), zl = zh + ZR * 16;
        const uint32_t acc = tbase + slot * 2 * MS;
#pragma unroll 4
        for (int ks = 0; ks < KL / 16; ++ks) {     // K = 16 per MMA: two 8-element chunks
          const uint64_t azh = make_sdesc(zh + ks * 256, 128, 128, LAYOUT_NONE);
          const uint64_t azl = make_sdesc(zl + ks * 256, 128, 128, LAYOUT_NONE);
          const uint64_t bd = make_sdesc(bc + ks * 2 * 2 * MS * 16, 2 * MS * 16, 128, LAYOUT_NONE);
          mma_f16_w(acc, azh, bd, idesc2, ks > 0);           // [hi.hi | hi.lo]
          mma_f16_w(acc + MS, azl, bd, idesc, 1);           // corr += lo.hi
        }
        mma_commit_w(&z_empty[slot]);
        mma_commit_w(&tfull[slot]);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..5)
    const int q = warp & 3, row = q * 32 + lane;
    const bool leader = (warp == 2 && lane == 0);
    // channels whose output parts are produced at the head (Ne - d == Kc, R24-R26) write them
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
      mbar_wait_u(&sc_full[i & 3], (uint32_t)((i >> 2) & 1));
      tc_fence_after();
      const float ti = tile_inv[i & 3];
      float v[MS], vc[MS];
      const uint32_t tacc = tbase + ((uint32_t)(q * 32) << 16) + slot * 2 * MS;
#pragma unroll
      for (int c0 = 0; c0 < MS; c0 += 16) tmem_ld16(tacc + c0, v + c0);
#pragma unroll
      for (int c0 = 0; c0 < MS; c0 += 16) tmem_ld16(tacc + MS + c0, vc + c0);
#pragma unroll
      for (int n = 0; n < MS; ++n) v[n] = (v[n] + vc[n]) * col_inv[n] * ti;   // main + corr, unscaled (exact)
      tc_fence_before();
      mbar_arrive(&tempty[slot]);
      if (to_parts) {                             // the 2^(depth+1) output parts instead of v
        const int64_t l = (tile_begin + i) * TM + row;
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
#pragma unroll
      for (int h = 0; h < 2; ++h) {               // two SW128 halves of 32 fp32 columns
        if (leader) bulk_wait_read0();            // the previous store has read the staging
        named_sync_h(1, 128);
        uint8_t* rrow = reinterpret_cast<uint8_t*>(Stg) + row * 128;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          *reinterpret_cast<float4*>(rrow + ((cc ^ (row & 7)) * 16)) =
              make_float4(v[32 * h + 4 * cc], v[32 * h + 4 * cc + 1], v[32 * h + 4 * cc + 2], v[32 * h + 4 * cc + 3]);
        fence_async_smem();
        named_sync_h(1, 128);
        if (leader) {
          tma_store_3d_h(&vmap, Stg, 32 * h, (int)((tile_begin + i) * TM), seq);
          bulk_commit_h();
        }
      }
    }
    if (leader) bulk_wait0();
  }
  __syncthreads();
  if (warp == 1) tmem_dealloc<4 * MS>(tbase);
}

int launch_bank_head_ws(int m, const BankHeadArg& a, int64_t n_seq_total, cudaStream_t st) {
  if (m != 64) return CASC_ERR_UNSUPPORTED;
  if (a.n_list <= 0) return CASC_OK;
  if (a.n_list * (int64_t)a.batch > 65535) return CASC_ERR_UNSUPPORTED;
  CUtensorMap vmap;
  if (!map3d(&vmap, a.V, true, 64, a.L, n_seq_total, TM)) return CASC_ERR_CUDA;
  const size_t smem = 1024 + (size_t)(TM * 32 + 2 * 264) * sizeof(float) + (size_t)(2 * KL * 64 + 2 * 2 * ZR * 8) * 2;
  if (cudaFuncSetAttribute(bank_head_ws_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return CASC_ERR_CUDA;
  const int64_t ntiles = ceil_div(a.L, TM);
  dim3 grid((unsigned)ceil_div(ntiles, a.tiles_per_cta), (unsigned)(a.n_list * a.batch));
  bank_head_ws_kernel<64><<<grid, 192, smem, st>>>(vmap, a);
  CASC_LAUNCHED();
  return CASC_OK;
}

}  // namespace casc
