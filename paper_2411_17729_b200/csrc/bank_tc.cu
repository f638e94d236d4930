// Bank of SISO channels (HiPPO example) on the sm_100a tensor cores.
//
// Per channel c with effective order Ne (stages k = 0..Ne) the path is
//   head  (a2+a3)  v^(Kc)_l = sum_{j < 2^Kc} (Abar^j Bbar) u_{l-j},  Kc = min(7, Ne)
//                  -- the first Kc stages of the cascade applied to v^(0) = Bbar u, written in
//                  the expanded form of their product prod_{n<Kc} (I + (z^-1 Abar)^(2^n)) =
//                  sum_{j<2^Kc} (z^-1 Abar)^j; one K = 128 GEMM per 128-step tile
//                  whose A operand (the Toeplitz matrix u_{l-j}) is a 4 KB shared-memory buffer.
//   stage (a4)     v^(k+1)_l = v^(k)_l + Abar^(2^k) v^(k)_{l-2^k},  k = Kc .. Ne-1 (2^k >= 128)
//   tail  (a5)     y_l = C v_l + (C Abar^(2^Ne)) v_{l-2^Ne} + D u_l   (stage Ne fused with y)
// fp32 accuracy from tcgen05 kind::tf32 with 3 products (hi.hi + lo.hi + hi.lo): the tensor
// core ignores the low 13 mantissa bits of an fp32 operand (truncation, checked by
// tests/test_gpu_tcgen05.py), so a raw fp32 tile IS its tf32 "hi" part and only
// lo = x - trunc(x) (exact in fp32) is materialised.
//
// Shared-memory operand layout: K-major, no swizzle; element (row r, k) at
//   (k/4)*LBO + r*16 + (k%4)*4,  SBO = 128 B (8 rows x 16 B), LBO = rows*16 B,
// linear in r, which lets a descriptor start at any row (used for the Toeplitz operand).
#include "common.cuh"
#include "kernels.cuh"
#include "sm100.cuh"
#include "bank_tc.cuh"

namespace casc {
using namespace sm100;

__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
__device__ __forceinline__ float tf32_lo(float x) { return x - tf32_trunc(x); }

template <int MS>
struct TmemCols {
  static constexpr int value = MS < 32 ? 32 : MS;
};

// ============================================================================ head
// grid.x: tile groups; grid.y: (list index) * batch + b. 128 threads.
template <int MS>
__global__ void __launch_bounds__(128) bank_head_kernel(BankHeadArg a) {
  constexpr int TM = 128, KL = 128;                   // time rows per tile, lags
  constexpr int BCH = KL / 4;                         // 16-B chunks along K (lags) = 32
  extern __shared__ __align__(1024) uint8_t smem[];
  float* Bhi = reinterpret_cast<float*>(smem);               // [BCH][MS][4]
  float* Blo = Bhi + KL * MS;
  float* Zhi = Blo + KL * MS;                                 // [256][4]
  float* Zlo = Zhi + 256 * 4;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid / 32;
  const int li = blockIdx.y / a.batch, b = blockIdx.y % a.batch;
  const int c = a.sys_list[li];
  const int64_t seq = (int64_t)c * a.batch + b;
  const float* u = a.u + seq * a.L;
  float* V = a.V + seq * a.L * MS;

  // B operand image: Kr^T (n = state, k' = 127 - lag), hi and lo, row-major in global
  const float* kh = a.krT + (int64_t)c * 2 * MS * KL;
  const float* kl = kh + MS * KL;
  for (int e = tid; e < MS * BCH; e += 128) {
    const int n = e / BCH, ch = e % BCH;
    const float4 h = *reinterpret_cast<const float4*>(kh + n * KL + ch * 4);
    const float4 l = *reinterpret_cast<const float4*>(kl + n * KL + ch * 4);
    *reinterpret_cast<float4*>(Bhi + (ch * MS + n) * 4) = h;
    *reinterpret_cast<float4*>(Blo + (ch * MS + n) * 4) = l;
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
  const int64_t ntiles = (a.L + TM - 1) / TM;
  const int64_t tile_begin = (int64_t)blockIdx.x * a.tiles_per_cta;
  const int64_t tile_end = min(ntiles, tile_begin + a.tiles_per_cta);
  uint32_t phase = 0;

  for (int64_t tile = tile_begin; tile < tile_end; ++tile) {
    const int64_t t0 = tile * TM;
    // Z-row w = (u[t0-127+w+i], i = 0..3), w = 0..251; the A operand row r, chunk c' is Z-row r+4c'
    for (int w = tid; w < 252; w += 128) {
      float z[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t t = t0 - (KL - 1) + w + i;
        z[i] = (t >= 0 && t < a.L) ? u[t] : 0.f;
      }
      *reinterpret_cast<float4*>(Zhi + w * 4) = make_float4(z[0], z[1], z[2], z[3]);
      *reinterpret_cast<float4*>(Zlo + w * 4) = make_float4(tf32_lo(z[0]), tf32_lo(z[1]), tf32_lo(z[2]), tf32_lo(z[3]));
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t zh = smem_u32(Zhi), zl = smem_u32(Zlo), bh = smem_u32(Bhi), bl = smem_u32(Blo);
#pragma unroll 4
      for (int ks = 0; ks < KL / 8; ++ks) {
        const uint64_t azh = make_sdesc(zh + ks * 128, 64, 128, LAYOUT_NONE);
        const uint64_t azl = make_sdesc(zl + ks * 128, 64, 128, LAYOUT_NONE);
        const uint64_t bdh = make_sdesc(bh + ks * 2 * MS * 16, MS * 16, 128, LAYOUT_NONE);
        const uint64_t bdl = make_sdesc(bl + ks * 2 * MS * 16, MS * 16, 128, LAYOUT_NONE);
        mma_tf32(tacc, azh, bdh, idesc, ks > 0);
        mma_tf32(tacc, azl, bdh, idesc, 1);
        mma_tf32(tacc, azh, bdl, idesc, 1);
      }
      mma_commit(&bar);
    }
    mbar_wait(&bar, phase);
    phase ^= 1;
    tc_fence_after();
    const int64_t row = t0 + tid;
    float* out = V + row * MS;
#pragma unroll
    for (int c0 = 0; c0 < MS; c0 += 16) {
      float v[16];
      tmem_ld16(tacc + ((uint32_t)(warp * 32) << 16) + c0, v);
      if (row < a.L) {
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(out + c0 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
    }
    tc_fence_before();
    __syncthreads();
  }
  if (warp == 0) tmem_dealloc<TmemCols<MS>::value>(tacc);
}

// ============================================================================ streaming stage
// v_dst[l] = v_src[l] + P_k v_src[l - 2^k], 2^k >= 128 (tile-aligned shift). grid as the head.
template <int MS>
__global__ void __launch_bounds__(128) bank_stage_kernel(BankStageArg a) {
  constexpr int TM = 128, CH = MS / 4;
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
  const int64_t ntiles = (a.L + TM - 1) / TM;
  const int64_t tile_begin = (int64_t)blockIdx.x * a.tiles_per_cta;
  const int64_t tile_end = min(ntiles, tile_begin + a.tiles_per_cta);
  uint32_t phase = 0;

  for (int64_t tile = tile_begin; tile < tile_end; ++tile) {
    const int64_t t0 = tile * TM, src0 = t0 - shift;
    const int64_t row = t0 + tid;
    // self row of this thread (epilogue operand), issued early
    float self[MS];
    if (row < a.L) {
#pragma unroll
      for (int i = 0; i < MS; i += 4) {
        const float4 v = *reinterpret_cast<const float4*>(Vs + row * MS + i);
        self[i] = v.x; self[i + 1] = v.y; self[i + 2] = v.z; self[i + 3] = v.w;
      }
    }
    if (src0 < 0) {                                  // l < 2^k: column unchanged
      if (row < a.L) {
#pragma unroll
        for (int i = 0; i < MS; i += 4)
          *reinterpret_cast<float4*>(Vd + row * MS + i) = make_float4(self[i], self[i + 1], self[i + 2], self[i + 3]);
      }
      continue;
    }
    // shifted tile rows [src0, src0+128) (always inside [0, L) since src0 + 127 < t0 <= L - 1).
    // A warp moves 8 rows x 4 chunks (8 x 64 contiguous bytes) per step; the smem side writes
    // 4 runs of 128 contiguous bytes (conflict-free).
    for (int e = tid; e < TM * CH; e += 128) {
      const int rblk = e / (8 * CH);                 // group of 8 rows
      const int rem = e % (8 * CH);
      const int ch = rem / 8, r = rblk * 8 + rem % 8;
      const float4 v = *reinterpret_cast<const float4*>(Vs + (src0 + r) * MS + ch * 4);
      *reinterpret_cast<float4*>(Ahi + (ch * TM + r) * 4) = v;
      *reinterpret_cast<float4*>(Alo + (ch * TM + r) * 4) =
          make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
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
    mbar_wait(&bar, phase);
    phase ^= 1;
    tc_fence_after();
#pragma unroll
    for (int c0 = 0; c0 < MS; c0 += 16) {
      float v[16];
      tmem_ld16(tacc + ((uint32_t)(warp * 32) << 16) + c0, v);
      if (row < a.L) {
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(Vd + row * MS + c0 + i) =
              make_float4(self[c0 + i] + v[i], self[c0 + i + 1] + v[i + 1], self[c0 + i + 2] + v[i + 2],
                          self[c0 + i + 3] + v[i + 3]);
      }
    }
    tc_fence_before();
    __syncthreads();
  }
  if (warp == 0) tmem_dealloc<TmemCols<MS>::value>(tacc);
}

// ============================================================================ tail
// y_l = C v_l + (C P_Ne) v_{l - 2^Ne} + D u_l ; thread per time step. grid.y = channel*batch.
template <int MS>
__global__ void __launch_bounds__(128) bank_tail_kernel(BankTailArg a) {
  __shared__ float cs[MS], ws[MS];
  const int c = blockIdx.y / a.batch, b = blockIdx.y % a.batch;
  const int64_t seq = (int64_t)c * a.batch + b;
  if (threadIdx.x < MS) {
    cs[threadIdx.x] = a.cvec[(int64_t)c * MS + threadIdx.x];
    ws[threadIdx.x] = a.wvec[(int64_t)c * MS + threadIdx.x];
  }
  __syncthreads();
  const float* V = (a.parity[c] ? a.Vb : a.Va) + seq * a.L * MS;
  const int64_t shift = (int64_t)1 << a.Neff[c];
  const float dc = a.d ? a.d[c] : 0.f;
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= a.L) return;
  float acc = dc * a.u[seq * a.L + l];
  const float* v0 = V + l * MS;
#pragma unroll
  for (int i = 0; i < MS; i += 4) {
    const float4 v = *reinterpret_cast<const float4*>(v0 + i);
    acc = fmaf(cs[i], v.x, acc); acc = fmaf(cs[i + 1], v.y, acc);
    acc = fmaf(cs[i + 2], v.z, acc); acc = fmaf(cs[i + 3], v.w, acc);
  }
  if (l - shift >= 0) {
    const float* v1 = V + (l - shift) * MS;
#pragma unroll
    for (int i = 0; i < MS; i += 4) {
      const float4 v = *reinterpret_cast<const float4*>(v1 + i);
      acc = fmaf(ws[i], v.x, acc); acc = fmaf(ws[i + 1], v.y, acc);
      acc = fmaf(ws[i + 2], v.z, acc); acc = fmaf(ws[i + 3], v.w, acc);
    }
  }
  a.y[seq * a.L + l] = acc;
}

// ============================================================================ derived data
// Kr64 [n][MS][128] float64 Krylov columns; column 0 = Bbar, the rest filled by dgemm levels.
__global__ void kr_init_kernel(const double* Bbar, double* Kr, int n, int ms) {
  const int64_t tot = (int64_t)n * ms * 128;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = e / (ms * 128), r = (e / 128) % ms, j = e % 128;
    Kr[e] = (j == 0) ? Bbar[s * ms + r] : 0.0;
  }
}
// krT32[s][0|1][n][k'] = hi | lo of Kr64[s][n][127 - k'], zero for lags >= 2^Kc[s]
__global__ void kr_split_kernel(const double* Kr, const int* Kc, float* krT, int n, int ms) {
  const int64_t tot = (int64_t)n * ms * 128;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = e / (ms * 128), r = (e / 128) % ms, kp = e % 128;
    const int j = 127 - (int)kp;
    const double v = (j < (1 << Kc[s])) ? Kr[(s * ms + r) * 128 + j] : 0.0;
    const float hi = tf32_rna((float)v);
    const float lo = tf32_rna((float)(v - (double)hi));
    float* base = krT + s * 2 * ms * 128;
    base[r * 128 + kp] = hi;
    base[ms * 128 + r * 128 + kp] = lo;
  }
}

int launch_kr_init(const double* Bbar, double* Kr, int n, int ms, cudaStream_t st) {
  const int64_t tot = (int64_t)n * ms * 128;
  kr_init_kernel<<<(int)std::min<int64_t>(ceil_div(tot, 256), 148 * 8), 256, 0, st>>>(Bbar, Kr, n, ms);
  CASC_LAUNCHED();
  return CASC_OK;
}
int launch_kr_split(const double* Kr, const int* Kc, float* krT, int n, int ms, cudaStream_t st) {
  const int64_t tot = (int64_t)n * ms * 128;
  kr_split_kernel<<<(int)std::min<int64_t>(ceil_div(tot, 256), 148 * 8), 256, 0, st>>>(Kr, Kc, krT, n, ms);
  CASC_LAUNCHED();
  return CASC_OK;
}

// ============================================================================ launchers
template <int MS>
static int head_launch(const BankHeadArg& a, cudaStream_t st) {
  const size_t smem = (size_t)(2 * 128 * MS + 2 * 256 * 4) * sizeof(float);
  cudaFuncSetAttribute(bank_head_kernel<MS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t ntiles = ceil_div(a.L, 128);
  dim3 grid((unsigned)ceil_div(ntiles, a.tiles_per_cta), (unsigned)(a.n_list * a.batch));
  bank_head_kernel<MS><<<grid, 128, smem, st>>>(a);
  CASC_LAUNCHED();
  return CASC_OK;
}
template <int MS>
static int stage_launch(const BankStageArg& a, cudaStream_t st) {
  const size_t smem = (size_t)(2 * MS * MS + 2 * 128 * MS) * sizeof(float);
  cudaFuncSetAttribute(bank_stage_kernel<MS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t ntiles = ceil_div(a.L, 128);
  dim3 grid((unsigned)ceil_div(ntiles, a.tiles_per_cta), (unsigned)(a.n_list * a.batch));
  bank_stage_kernel<MS><<<grid, 128, smem, st>>>(a);
  CASC_LAUNCHED();
  return CASC_OK;
}
template <int MS>
static int tail_launch(const BankTailArg& a, cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(a.L, 128), (unsigned)(a.n_ch * a.batch));
  bank_tail_kernel<MS><<<grid, 128, 0, st>>>(a);
  CASC_LAUNCHED();
  return CASC_OK;
}

bool bank_tc_supported(int m) { return m == 16 || m == 32 || m == 64; }

int launch_bank_head(int m, const BankHeadArg& a, cudaStream_t st) {
  if (a.n_list <= 0) return CASC_OK;
  if (a.n_list * (int64_t)a.batch > 65535) return CASC_ERR_UNSUPPORTED;
  switch (m) {
    case 16: return head_launch<16>(a, st);
    case 32: return head_launch<32>(a, st);
    case 64: return head_launch<64>(a, st);
  }
  return CASC_ERR_UNSUPPORTED;
}
int launch_bank_stage(int m, const BankStageArg& a, cudaStream_t st) {
  if (a.n_list <= 0) return CASC_OK;
  if (a.n_list * (int64_t)a.batch > 65535) return CASC_ERR_UNSUPPORTED;
  switch (m) {
    case 16: return stage_launch<16>(a, st);
    case 32: return stage_launch<32>(a, st);
    case 64: return stage_launch<64>(a, st);
  }
  return CASC_ERR_UNSUPPORTED;
}
int launch_bank_tail(int m, const BankTailArg& a, cudaStream_t st) {
  if (a.n_ch * (int64_t)a.batch > 65535) return CASC_ERR_UNSUPPORTED;
  switch (m) {
    case 16: return tail_launch<16>(a, st);
    case 32: return tail_launch<32>(a, st);
    case 64: return tail_launch<64>(a, st);
  }
  return CASC_ERR_UNSUPPORTED;
}

}  // namespace casc
