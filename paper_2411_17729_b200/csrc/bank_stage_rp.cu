// Streaming cascade stage of the SISO bank (register-prefetch variant, the default):
//   v_dst[l] = v_src[l] + Abar^(2^k) v_src[l - 2^k], 2^k >= 128
// 128 threads, two CTAs per SM. Per 128-step tile: the shifted tile is loaded (8 rows x 64 B
// per warp instruction) into registers one tile ahead, stored to shared memory as raw fp32
// (= tf32 hi by truncation) and lo = x - trunc(x), 3xTF32 tcgen05.mma (M=128, N=K=MS) into
// TMEM, epilogue adds the thread's own row and writes through a warp-private swizzled slab.
#include "common.cuh"
#include "sm100.cuh"
#include "bank_tc.cuh"
#include "bank_common.cuh"

namespace casc {
using namespace sm100;

// ============================================================================ streaming stage
// v_dst[l] = v_src[l] + P_k v_src[l - 2^k], 2^k >= 128 (tile-aligned shift). grid as the head.
// Rows l < 2^k are copies; for k > first streaming stage the destination already holds
// v^(k-1) = v^(k+1) on l < 2^(k-1), so only [copy_from, 2^k) is copied.
template <int MS>
__global__ void __launch_bounds__(128) bank_stage_rp_kernel(BankStageArg a) {
  constexpr int TM = 128, CH = MS / 4, NLD = TM * CH / 128;
  extern __shared__ __align__(1024) uint8_t smem[];
  float* Phi = reinterpret_cast<float*>(smem);     // [CH][MS][4]
  float* Plo = Phi + MS * MS;
  float* Ahi = Plo + MS * MS;                      // [CH][TM][4] raw fp32 (= tf32 hi by truncation)
  float* Alo = Ahi + TM * MS;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int li = blockIdx.y / a.batch, b = blockIdx.y % a.batch;
  const int c = a.sys_list[li];
  const int64_t seq = (int64_t)c * a.batch + b;
  const float* Vs = a.Vs + seq * a.L * MS;
  float* Vd = a.Vd + seq * a.L * MS;
  const int64_t shift = (int64_t)1 << a.k;

  const int64_t ntiles = (a.L + TM - 1) / TM;
  const int64_t tile_begin = (int64_t)blockIdx.x * a.tiles_per_cta;
  const int64_t tile_end = ntiles < tile_begin + a.tiles_per_cta ? ntiles : tile_begin + a.tiles_per_cta;
  // tiles entirely below copy_from need no work at all
  const int64_t first_needed = a.copy_from / TM;
  const int64_t tb = tile_begin > first_needed ? tile_begin : first_needed;
  if (tb >= tile_end) return;

  const float* ph = a.P + ((int64_t)c * a.slots + a.k) * 2 * MS * MS;
  const float* pl = ph + MS * MS;
  for (int e = tid; e < MS * CH; e += 128) {
    const int n = e / CH, ch = e % CH;
    *reinterpret_cast<float4*>(Phi + (ch * MS + n) * 4) = *reinterpret_cast<const float4*>(ph + n * MS + ch * 4);
    *reinterpret_cast<float4*>(Plo + (ch * MS + n) * 4) = *reinterpret_cast<const float4*>(pl + n * MS + ch * 4);
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<TmemCols<MS>::value>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tacc = tmem_base;
  const uint32_t idesc = make_idesc(FMT_TF32, TM, MS);
  uint32_t phase = 0;

  float4 areg[NLD];
  // self rows of this warp (rows 32*warp .. +31 of the tile) in the warp-coalesced mapping:
  // sweep it covers RPS consecutive rows, lane -> (row it*RPS + lane/CH, 16-B chunk lane%CH)
  constexpr int RPS = 32 / CH;
  float4 s4[CH];
  // shifted tile rows [src0, src0+128): a warp moves 8 rows x 4 chunks (8 x 64 B) per load
  auto load_a = [&](int64_t src0) {
#pragma unroll
    for (int it = 0; it < NLD; ++it) {
      const int e = it * 128 + tid;
      const int rem = e % (8 * CH), ch = rem / 8, r = (e / (8 * CH)) * 8 + rem % 8;
      areg[it] = __ldg(reinterpret_cast<const float4*>(Vs + (src0 + r) * MS + ch * 4));
    }
  };
  auto load_s = [&](int64_t t0) {
    const int64_t r0 = t0 + warp * 32;
#pragma unroll
    for (int it = 0; it < CH; ++it) {
      const int64_t row = r0 + it * RPS + lane / CH;
      s4[it] = row < a.L ? __ldg(reinterpret_cast<const float4*>(Vs + row * MS + (lane % CH) * 4))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  // store this warp's 32 rows: optional per-thread-row values v (TMEM lane order) are first
  // transposed through the warp's swizzled smem slab, then added to s4 and written coalesced
  auto store_rows = [&](float* slab, const float* v, int64_t r0, int valid) {
    if (v) {
#pragma unroll
      for (int j = 0; j < CH; ++j)
        *reinterpret_cast<float4*>(slab + lane * MS + ((j ^ (lane % CH)) * 4)) =
            make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      __syncwarp();
    }
#pragma unroll
    for (int it = 0; it < CH; ++it) {
      const int r = it * RPS + lane / CH, j = lane % CH;
      float4 o = s4[it];
      if (v) {
        const float4 p = *reinterpret_cast<const float4*>(slab + r * MS + ((j ^ (r % CH)) * 4));
        o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
      }
      if (r < valid) *reinterpret_cast<float4*>(Vd + (r0 + r) * MS + j * 4) = o;
    }
    __syncwarp();
  };
  if (tb * TM - shift >= 0) load_a(tb * TM - shift);
  load_s(tb * TM);

  for (int64_t tile = tb; tile < tile_end; ++tile) {
    const int64_t t0 = tile * TM, src0 = t0 - shift;
    const int64_t r0 = t0 + warp * 32;
    const int64_t rem_rows = a.L - r0;
    const int valid = (int)(rem_rows < 0 ? 0 : (rem_rows < 32 ? rem_rows : 32));
    const bool has_next = tile + 1 < tile_end;
    if (src0 < 0) {                                  // l < 2^k: column unchanged
      store_rows(nullptr, nullptr, r0, valid);
      if (has_next) {
        if (src0 + TM >= 0) load_a(src0 + TM);
        load_s(t0 + TM);
      }
      continue;
    }
#pragma unroll
    for (int it = 0; it < NLD; ++it) {
      const int e = it * 128 + tid;
      const int rem = e % (8 * CH), ch = rem / 8, r = (e / (8 * CH)) * 8 + rem % 8;
      const float4 v = areg[it], h = tf32_hi4(v);
      *reinterpret_cast<float4*>(Ahi + (ch * TM + r) * 4) = h;
      *reinterpret_cast<float4*>(Alo + (ch * TM + r) * 4) = tf32_lo4(v, h);
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t ah = smem_u32(Ahi), al = smem_u32(Alo), bh = smem_u32(Phi), bl = smem_u32(Plo);
#pragma unroll
      for (int ks = 0; ks < MS / 8; ++ks) {
        const uint64_t dah = make_sdesc(ah + ks * 2 * TM * 16, TM * 16, 128, LAYOUT_NONE);
        const uint64_t dal = make_sdesc(al + ks * 2 * TM * 16, TM * 16, 128, LAYOUT_NONE);
        const uint64_t dbh = make_sdesc(bh + ks * 2 * MS * 16, MS * 16, 128, LAYOUT_NONE);
        const uint64_t dbl = make_sdesc(bl + ks * 2 * MS * 16, MS * 16, 128, LAYOUT_NONE);
        mma_tf32(tacc, dah, dbh, idesc, ks > 0);
        mma_tf32(tacc, dal, dbh, idesc, 1);
        mma_tf32(tacc, dah, dbl, idesc, 1);
      }
      mma_commit(&bar);
    }
    if (has_next) load_a(t0 + TM - shift);           // prefetch (src0 >= 0 implies next >= 0)
    mbar_wait(&bar, phase);
    phase ^= 1;
    tc_fence_after();
    float v[MS];
#pragma unroll
    for (int c0 = 0; c0 < MS; c0 += 16) tmem_ld16(tacc + ((uint32_t)(warp * 32) << 16) + c0, v + c0);
    tc_fence_before();
    store_rows(Ahi + warp * 32 * MS, v, r0, valid);   // slab in Ahi: free once the MMA completed
    if (has_next) load_s(t0 + TM);
    __syncthreads();
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc<TmemCols<MS>::value>(tacc);
}


template <int MS>
static int rp_launch(const BankStageArg& a, cudaStream_t st) {
  const size_t smem = (size_t)(2 * MS * MS + 2 * 128 * MS) * sizeof(float);
  if (cudaFuncSetAttribute(bank_stage_rp_kernel<MS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return CASC_ERR_CUDA;
  const int64_t ntiles = ceil_div(a.L, 128);
  dim3 grid((unsigned)ceil_div(ntiles, a.tiles_per_cta), (unsigned)(a.n_list * a.batch));
  bank_stage_rp_kernel<MS><<<grid, 128, smem, st>>>(a);
  CASC_LAUNCHED();
  return CASC_OK;
}

int launch_bank_stage_rp(int m, const BankStageArg& a, cudaStream_t st) {
  if (a.n_list <= 0) return CASC_OK;
  if (a.n_list * (int64_t)a.batch > 65535) return CASC_ERR_UNSUPPORTED;
  switch (m) {
    case 16: return rp_launch<16>(a, st);
    case 32: return rp_launch<32>(a, st);
    case 64: return rp_launch<64>(a, st);
  }
  return CASC_ERR_UNSUPPORTED;
}

}  // namespace casc
