// Streaming cascade stage of the SISO bank, warp-specialized and persistent (sm_100a):
//
//   v_dst[l] = v_src[l] + Abar^(2^k) v_src[l - 2^k], 2^k >= 128
//
// One CTA per SM (256 threads) walks tiles of 128 time steps of one sequence at a time
// (blocks of G tiles dealt round-robin over the grid so that the chip sweeps the sequences in
// order and the shifted reads at l - 2^k hit L2):
//   warps 4-7 (producer): cp.async 3-deep ring of the shifted fp32 tile (raw bits = tf32 hi),
//                         lo = x - trunc(x) split, tcgen05.mma issue (3xTF32, M=128 N=MS K=MS)
//                         into one of two TMEM accumulators, tcgen05.commit -> mma_done[acc]
//   warps 0-3 (epilogue): cp.async double-buffered self tile into a row-swizzled slab, TMEM
//                         drain (lane = time row), v += acc in place, arrive acc_free[acc],
//                         512-byte coalesced stores of the finished rows.
// Tiles l < 2^k are copies (no MMA; an empty commit keeps the barrier protocol uniform); tiles
// entirely below copy_from are skipped because the destination already holds their values.
#include "common.cuh"
#include "sm100.cuh"
#include "bank_tc.cuh"

namespace casc {
using namespace sm100;

namespace {

constexpr int TM = 128;          // time rows per tile
constexpr int NS = 3;            // shifted-tile ring depth
constexpr int GT = 16;           // tiles per work block

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Deterministic walk over this CTA's tiles (both warp groups run their own copy).
struct TileWalk {
  int64_t q, t, t_hi;            // current block, tile, block end
  int64_t nblk, nblocks, ntiles, first_needed;
  bool valid;
  __device__ void init(int64_t ntiles_, int64_t nseq, int64_t first_needed_) {
    ntiles = ntiles_;
    first_needed = first_needed_;
    nblk = (ntiles + GT - 1) / GT;
    nblocks = nblk * nseq;
    q = blockIdx.x;
    t = -1;
    t_hi = -1;
    advance();
  }
  __device__ void advance() {
    ++t;
    while (true) {
      if (q >= nblocks) { valid = false; return; }
      const int64_t blk = q % nblk;
      const int64_t lo = max(blk * GT, first_needed);
      t_hi = min(blk * GT + GT, ntiles);
      if (t < lo) t = lo;
      if (t < t_hi) { valid = true; return; }
      q += gridDim.x;
      t = -1;
    }
  }
  __device__ int64_t seq_index() const { return q / nblk; }   // index into (list, batch)
};

}  // namespace

template <int MS>
__global__ void __launch_bounds__(256, 1) bank_stage_ws_kernel(BankStageArg a) {
  constexpr int CH = MS / 4;                  // 16-B chunks per row
  constexpr int TCOLS = (2 * MS) < 32 ? 32 : 2 * MS;
  extern __shared__ __align__(1024) uint8_t smem[];
  float* Phi = reinterpret_cast<float*>(smem);          // [CH][MS][4]
  float* Plo = Phi + MS * MS;
  float* Araw = Plo + MS * MS;                          // [NS][CH][TM][4]
  float* Alo = Araw + NS * TM * MS;                     // [CH][TM][4]
  float* Slf = Alo + TM * MS;                           // [2][TM][MS] row-swizzled
  __shared__ uint64_t mma_done[2], acc_free[2];
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int64_t shift = (int64_t)1 << a.k;
  const int64_t ntiles = (a.L + TM - 1) / TM;
  const int64_t nseq = (int64_t)a.n_list * a.batch;

  if (tid == 0) {
    mbar_init(&mma_done[0], 1);
    mbar_init(&mma_done[1], 1);
    mbar_init(&acc_free[0], 128);
    mbar_init(&acc_free[1], 128);
    fence_mbar_init();
  }
  if (warp == 4) tmem_alloc<TCOLS>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;

  if (warp >= 4) {
    // =================================================================== producer
    const int pt = tid - 128;
    const uint32_t idesc = make_idesc(FMT_TF32, TM, MS);
    TileWalk cur, ld;
    cur.init(ntiles, nseq, a.copy_from / TM);
    ld.init(ntiles, nseq, a.copy_from / TM);
    auto seq_ptr = [&](int64_t si) {
      const int c = a.sys_list[si / a.batch];
      return a.Vs + ((int64_t)c * a.batch + si % a.batch) * a.L * MS;
    };
    // issue the shifted-tile loads of walk position `w` into ring slot `slot`
    auto issue_load = [&](const TileWalk& w, int slot) {
      if (w.valid) {
        const int64_t src0 = w.t * TM - shift;
        if (src0 >= 0) {
          const float* Vs = seq_ptr(w.seq_index());
          float* dst = Araw + slot * TM * MS;
#pragma unroll
          for (int it = 0; it < TM * CH / 128; ++it) {
            const int e = it * 128 + pt;
            const int rem = e % (8 * CH), ch = rem / 8, r = (e / (8 * CH)) * 8 + rem % 8;
            cp_async16(dst + (ch * TM + r) * 4, Vs + (src0 + r) * MS + ch * 4);
          }
        }
      }
      cp_async_commit();
    };
    for (int s = 0; s < NS - 1; ++s) {
      issue_load(ld, s);
      ld.advance();
    }
    int cur_channel = -1;
    int64_t i = 0;
    for (; cur.valid; cur.advance(), ++i) {
      // tile i-1's MMAs must be done before its ring slot, Alo (and possibly P) are reused
      if (i >= 1) mbar_wait(&mma_done[(i - 1) & 1], ((i - 1) >> 1) & 1);
      issue_load(ld, (int)((i + NS - 1) % NS));
      ld.advance();
      const int64_t src0 = cur.t * TM - shift;
      const int c = a.sys_list[cur.seq_index() / a.batch];
      if (c != cur_channel) {                       // (re)load P_k of this channel
        const float* ph = a.P + ((int64_t)c * a.slots + a.k) * 2 * MS * MS;
        const float* pl = ph + MS * MS;
        for (int e = pt; e < MS * CH; e += 128) {
          const int ch = e / MS, n = e % MS;
          *reinterpret_cast<float4*>(Phi + (ch * MS + n) * 4) = __ldg(reinterpret_cast<const float4*>(ph + n * MS + ch * 4));
          *reinterpret_cast<float4*>(Plo + (ch * MS + n) * 4) = __ldg(reinterpret_cast<const float4*>(pl + n * MS + ch * 4));
        }
        fence_async_smem();                         // P is read by the tensor core (async proxy)
        cur_channel = c;
      }
      cp_async_wait<NS - 1>();                     // this thread's copies of tile i landed
      named_sync(1, 128);
      const bool mma = src0 >= 0;
      if (mma) {
        float* ar = Araw + (i % NS) * TM * MS;
        for (int e = pt; e < TM * CH; e += 128) {
          const float4 v = *reinterpret_cast<const float4*>(ar + e * 4), h = tf32_hi4(v);
          *reinterpret_cast<float4*>(ar + e * 4) = h;
          *reinterpret_cast<float4*>(Alo + e * 4) = tf32_lo4(v, h);
        }
        fence_async_smem();
      }
      named_sync(1, 128);
      if (pt == 0) {
        if (i >= 2) mbar_wait(&acc_free[i & 1], ((i - 2) >> 1) & 1);
        tc_fence_after();
        const uint32_t acc = tbase + (uint32_t)(i & 1) * MS;
        if (mma) {
          const uint32_t ah = smem_u32(Araw + (i % NS) * TM * MS), al = smem_u32(Alo);
          const uint32_t bh = smem_u32(Phi), bl = smem_u32(Plo);
#pragma unroll
          for (int ks = 0; ks < MS / 8; ++ks) {
            const uint64_t dah = make_sdesc(ah + ks * 2 * TM * 16, TM * 16, 128, LAYOUT_NONE);
            const uint64_t dal = make_sdesc(al + ks * 2 * TM * 16, TM * 16, 128, LAYOUT_NONE);
            const uint64_t dbh = make_sdesc(bh + ks * 2 * MS * 16, MS * 16, 128, LAYOUT_NONE);
            const uint64_t dbl = make_sdesc(bl + ks * 2 * MS * 16, MS * 16, 128, LAYOUT_NONE);
            mma_tf32(acc, dah, dbh, idesc, ks > 0);
            mma_tf32(acc, dal, dbh, idesc, 1);
            mma_tf32(acc, dah, dbl, idesc, 1);
          }
        }
        mma_commit(&mma_done[i & 1]);
      }
    }
    cp_async_wait<0>();
  } else {
    // =================================================================== epilogue
    TileWalk cur, ld;
    cur.init(ntiles, nseq, a.copy_from / TM);
    ld.init(ntiles, nseq, a.copy_from / TM);
    auto seq_off = [&](int64_t si) {
      const int c = a.sys_list[si / a.batch];
      return ((int64_t)c * a.batch + si % a.batch) * a.L * MS;
    };
    // cp.async this warp's 32 self rows of walk position `w` into slab slot `slot`
    auto issue_self = [&](const TileWalk& w, int slot) {
      if (w.valid) {
        const float* Vs = a.Vs + seq_off(w.seq_index());
        float* dst = Slf + slot * TM * MS + warp * 32 * MS;
        const int64_t r0 = w.t * TM + warp * 32;
#pragma unroll
        for (int it = 0; it < 32 / (32 / CH); ++it) {
          const int r = it * (32 / CH) + lane / CH, j = lane % CH;
          const bool ok = r0 + r < a.L;
          cp_async16_zfill(dst + r * MS + ((j ^ (r % CH)) * 4), Vs + (ok ? (r0 + r) * MS + j * 4 : 0), ok);
        }
      }
      cp_async_commit();
    };
    issue_self(ld, 0);
    ld.advance();
    int64_t i = 0;
    for (; cur.valid; cur.advance(), ++i) {
      issue_self(ld, (int)((i + 1) & 1));
      ld.advance();
      const int64_t src0 = cur.t * TM - shift;
      float* slab = Slf + (i & 1) * TM * MS + warp * 32 * MS;
      mbar_wait(&mma_done[i & 1], (i >> 1) & 1);
      tc_fence_after();
      cp_async_wait<1>();
      __syncwarp();
      if (src0 >= 0) {
        const uint32_t acc = tbase + ((uint32_t)(warp * 32) << 16) + (uint32_t)(i & 1) * MS;
        float* row = slab + lane * MS;
#pragma unroll
        for (int c0 = 0; c0 < MS; c0 += 16) {
          float v[16];
          tmem_ld16(acc + c0, v);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int j = c0 / 4 + q;
            float4* p = reinterpret_cast<float4*>(row + ((j ^ (lane % CH)) * 4));
            float4 s = *p;
            s.x += v[4 * q]; s.y += v[4 * q + 1]; s.z += v[4 * q + 2]; s.w += v[4 * q + 3];
            *p = s;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_free[i & 1]);
      __syncwarp();
      float* Vd = a.Vd + seq_off(cur.seq_index());
      const int64_t r0 = cur.t * TM + warp * 32;
#pragma unroll
      for (int it = 0; it < 32 / (32 / CH); ++it) {
        const int r = it * (32 / CH) + lane / CH, j = lane % CH;
        if (r0 + r < a.L)
          *reinterpret_cast<float4*>(Vd + (r0 + r) * MS + j * 4) =
              *reinterpret_cast<const float4*>(slab + r * MS + ((j ^ (r % CH)) * 4));
      }
      __syncwarp();
    }
    cp_async_wait<0>();
  }
  __syncthreads();
  if (warp == 4) tmem_dealloc<TCOLS>(tbase);
}

template <int MS>
static int ws_launch(const BankStageArg& a, cudaStream_t st) {
  const size_t smem = (size_t)(2 * MS * MS + NS * TM * MS + TM * MS + 2 * TM * MS) * sizeof(float);
  if (cudaFuncSetAttribute(bank_stage_ws_kernel<MS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return CASC_ERR_CUDA;
  const int64_t ntiles = ceil_div(a.L, TM);
  const int64_t nblocks = ceil_div(ntiles, GT) * (int64_t)a.n_list * a.batch;
  const int grid = (int)std::min<int64_t>(nblocks, 148);
  bank_stage_ws_kernel<MS><<<grid, 256, smem, st>>>(a);
  CASC_LAUNCHED();
  return CASC_OK;
}

int launch_bank_stage_ws(int m, const BankStageArg& a, cudaStream_t st) {
  if (a.n_list <= 0) return CASC_OK;
  switch (m) {
    case 16: return ws_launch<16>(a, st);
    case 32: return ws_launch<32>(a, st);
    case 64: return ws_launch<64>(a, st);
  }
  return CASC_ERR_UNSUPPORTED;
}

}  // namespace casc
