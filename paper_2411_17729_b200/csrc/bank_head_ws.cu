// Bank head (stages 0..Kc-1 with Bbar u, R22), warp-specialized (m = 64):
//
//   v^(Kc)_l = sum_{j < 128} (Abar^j Bbar) u_{l-j}     (the expanded product of PAPER.md:126)
//
// per 128-step tile one K = 128 GEMM (3xTF32: hi.hi + lo.hi + hi.lo) whose A operand, the
// Toeplitz matrix u_{l-j}, is a 4 KB shared-memory buffer Z read with LBO = 64 B (row r, K chunk
// c' = Z-row r + 4c'). The Krylov weights are stored hi and lo stacked along N ([K chunk][hi 64 |
// lo 64 rows]), so Z_hi x [B_hi | B_lo] is one N = 128 MMA writing hi.hi to the main and hi.lo to
// the correction accumulator, and Z_lo x B_hi (N = 64) adds to the correction: the MMAs read 14 KB
// of shared memory per K step instead of 18 KB (shared-memory bandwidth bounds this kernel).
// Roles (192 threads, two CTAs per SM):
//   warp 0     builds Z for the next tiles into a 2-slot ring (u staged through shared memory)
//   warp 1     issues the 32 MMAs of a tile into one of two TMEM accumulators (main | corr)
//   warps 2-5  drain TMEM (lane = time row) into a SWIZZLE_128B staging tile and TMA-store it
// Each CTA walks `tiles_per_cta` consecutive tiles of one sequence, so the Krylov weights
// (64 KB of hi/lo) are loaded once per CTA.
#include <cuda.h>

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
}  // namespace

template <int MS>
__global__ void __launch_bounds__(192, 2) bank_head_ws_kernel(const __grid_constant__ CUtensorMap vmap, BankHeadArg a) {
  static_assert(MS == 64, "TMA-store epilogue written for m = 64");
  constexpr int BCH = KL / 4;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps the shared state space (STS/LDS, not generic ST/LD)
  float* Stg = reinterpret_cast<float*>(smem);                 // [128 rows][32] SW128 half tile, 16 KB
  float* Bc = Stg + TM * 32;                                   // [BCH][hi MS | lo MS][4]
  float* Zb = Bc + 2 * KL * MS;                                // [2 slots][hi|lo][ZR][4]
  float* Us = Zb + 2 * 2 * ZR * 4;                             // [2 slots][264] u window
  __shared__ uint64_t z_full[2], z_empty[2], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid / 32, 0), lane = tid % 32;
  const int li = blockIdx.y / a.batch, b = blockIdx.y % a.batch;
  const int c = a.sys_list[li];
  const int seq = c * a.batch + b;
  const float* u = a.u + (int64_t)seq * a.L;

  const float* kh = a.krT + (int64_t)c * 2 * MS * KL;
  const float* kl = kh + MS * KL;
  for (int e = tid; e < MS * BCH; e += 192) {
    const int ch = e / MS, n = e % MS;
    *reinterpret_cast<float4*>(Bc + (ch * 2 * MS + n) * 4) = __ldg(reinterpret_cast<const float4*>(kh + n * KL + ch * 4));
    *reinterpret_cast<float4*>(Bc + (ch * 2 * MS + MS + n) * 4) = __ldg(reinterpret_cast<const float4*>(kl + n * KL + ch * 4));
  }
  fence_async_smem();
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&z_full[s], 32);
      mbar_init(&z_empty[s], 1);
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
    }
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
      mbar_arrive(&z_full[slot]);
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
      const uint32_t idesc = make_idesc(FMT_TF32, TM, MS), idesc2 = make_idesc(FMT_TF32, TM, 2 * MS);
      const uint32_t bc = smem_u32(Bc);
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
          const uint64_t bd = make_sdesc(bc + ks * 2 * 2 * MS * 16, 2 * MS * 16, 128, LAYOUT_NONE);
          mma_tf32_w(acc, azh, bd, idesc2, ks > 0);          // [hi.hi | hi.lo]
          mma_tf32_w(acc + MS, azl, bd, idesc, 1);          // corr += lo.hi
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
  const size_t smem = 1024 + (size_t)(TM * 32 + 2 * KL * 64 + 2 * 2 * ZR * 4 + 2 * 264) * sizeof(float);
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
