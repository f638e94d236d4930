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
#include <cuda_fp16.h>
#include "bank_common.cuh"

namespace casc {
using namespace sm100;

// ============================================================================ head
// grid.x: tile groups; grid.y: (list index) * batch + b. 128 threads (4 warps).
// Z and the TMEM accumulator are double-buffered: the MMA of tile i+1 runs while the
// epilogue drains tile i.
template <int MS>
__global__ void __launch_bounds__(128) bank_head_kernel(BankHeadArg a) {
  constexpr int TM = 128, KL = 128;                   // time rows per tile, lags
  constexpr int BCH = KL / 4;                         // 16-B chunks along K (lags) = 32
  constexpr int ZR = 256;                             // Z rows (252 used)
  extern __shared__ __align__(1024) uint8_t smem[];
  float* Bhi = reinterpret_cast<float*>(smem);        // [BCH][MS][4]
  float* Blo = Bhi + KL * MS;
  float* Zbuf = Blo + KL * MS;                        // [2 buf][hi|lo][ZR][4]
  float* Stg = Zbuf + 2 * 2 * ZR * 4;                 // [4 warps][32][MS] staging
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int li = blockIdx.y / a.batch, b = blockIdx.y % a.batch;
  const int c = a.sys_list[li];
  const int64_t seq = (int64_t)c * a.batch + b;
  const float* u = a.u + seq * a.L;
  float* V = a.V + seq * a.L * MS;

  const float* kh = a.krT + (int64_t)c * 2 * MS * KL;
  const float* kl = kh + MS * KL;
  for (int e = tid; e < MS * BCH; e += 128) {
    const int ch = e / MS, n = e % MS;                // consecutive threads -> consecutive smem chunks
    *reinterpret_cast<float4*>(Bhi + (ch * MS + n) * 4) = *reinterpret_cast<const float4*>(kh + n * KL + ch * 4);
    *reinterpret_cast<float4*>(Blo + (ch * MS + n) * 4) = *reinterpret_cast<const float4*>(kl + n * KL + ch * 4);
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  constexpr int TCOLS = TmemCols<2 * MS>::value;
  if (warp == 0) tmem_alloc<TCOLS>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  const uint32_t idesc = make_idesc(FMT_TF32, TM, MS);
  const int64_t ntiles = (a.L + TM - 1) / TM;
  const int64_t tile_begin = (int64_t)blockIdx.x * a.tiles_per_cta;
  const int64_t tile_end = min(ntiles, tile_begin + a.tiles_per_cta);
  const int nt = (int)(tile_end - tile_begin);

  // Z-row w = (u[t0-127+w+i], i = 0..3); A operand (row r, chunk c') = Z-row r + 4c'.
  // Thread tid owns Z-rows tid and tid+128; their u values are prefetched into registers one
  // tile ahead (load_u) so the global latency is off the critical path.
  float zr[2][4];
  auto load_u = [&](int i) {
    const int64_t t0 = (tile_begin + i) * TM;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t t = t0 - (KL - 1) + tid + 128 * h + q;
        zr[h][q] = (i < nt && t >= 0 && t < a.L) ? __ldg(u + t) : 0.f;
      }
  };
  auto build_z = [&](int i) {
    float* zh = Zbuf + (i & 1) * 2 * ZR * 4;
    float* zl = zh + ZR * 4;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int w = tid + 128 * h;
      const float4 z = make_float4(zr[h][0], zr[h][1], zr[h][2], zr[h][3]), zhi = tf32_hi4(z);
      *reinterpret_cast<float4*>(zh + w * 4) = zhi;
      *reinterpret_cast<float4*>(zl + w * 4) = tf32_lo4(z, zhi);
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t zhs = smem_u32(zh), zls = smem_u32(zl), bh = smem_u32(Bhi), bl = smem_u32(Blo);
      const uint32_t acc = tbase + (i & 1) * MS;
#pragma unroll 4
      for (int ks = 0; ks < KL / 8; ++ks) {
        const uint64_t azh = make_sdesc(zhs + ks * 128, 64, 128, LAYOUT_NONE);
        const uint64_t azl = make_sdesc(zls + ks * 128, 64, 128, LAYOUT_NONE);
        const uint64_t bdh = make_sdesc(bh + ks * 2 * MS * 16, MS * 16, 128, LAYOUT_NONE);
        const uint64_t bdl = make_sdesc(bl + ks * 2 * MS * 16, MS * 16, 128, LAYOUT_NONE);
        mma_tf32(acc, azh, bdh, idesc, ks > 0);
        mma_tf32(acc, azl, bdh, idesc, 1);
        mma_tf32(acc, azh, bdl, idesc, 1);
      }
      mma_commit(&bar[i & 1]);
    }
  };

  if (nt > 0) {
    load_u(0);
    build_z(0);
    load_u(1);
  }
  for (int i = 0; i < nt; ++i) {
    if (i + 1 < nt) {
      build_z(i + 1);
      load_u(i + 2);
    }
    mbar_wait(&bar[i & 1], (i >> 1) & 1);
    tc_fence_after();
    const int64_t t0 = (tile_begin + i) * TM;
    float v[MS];
#pragma unroll
    for (int c0 = 0; c0 < MS; c0 += 16)
      tmem_ld16(tbase + ((uint32_t)(warp * 32) << 16) + (i & 1) * MS + c0, v + c0);
    tc_fence_before();
    const int64_t r0 = t0 + warp * 32;
    warp_store_rows<MS>(Stg + warp * 32 * MS, v, V + r0 * MS, lane, (int)(a.L - r0 < 32 ? a.L - r0 : 32));
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc<TCOLS>(tbase);
}

// ============================================================================ tail
// y_l = C v_l + (C P_Ne) v_{l - 2^Ne} + D u_l. One warp per 32 consecutive time steps: each
// row (MS floats) is read by the whole warp as one coalesced load, per-lane partial dot
// products are reduced with a 31-shuffle transpose so lane i ends with y_{l0+i}.
template <int MS>
__global__ void __launch_bounds__(256) bank_tail_kernel(BankTailArg a) {
  constexpr int VPL = MS >= 32 ? MS / 32 : 1;         // values per lane
  constexpr int ACT = MS / VPL;                       // active lanes per row
  const int c = blockIdx.y / a.batch, b = blockIdx.y % a.batch;
  const int64_t seq = (int64_t)c * a.batch + b;
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  const float* V = (a.parity[c] ? a.Vb : a.Va) + seq * a.L * MS;
  const int64_t shift = (int64_t)1 << a.Neff[c];
  float cw[VPL], ww[VPL];
#pragma unroll
  for (int q = 0; q < VPL; ++q) {
    const int idx = lane * VPL + q;
    cw[q] = lane < ACT ? a.cvec[(int64_t)c * MS + idx] : 0.f;
    ww[q] = lane < ACT ? a.wvec[(int64_t)c * MS + idx] : 0.f;
  }
  const float dc = a.d[c];
  const int64_t l0 = ((int64_t)blockIdx.x * 8 + warp) * 32;
  if (l0 >= a.L) return;
  // all 64 row loads of the warp are issued before any use (clamped addresses, masked weights)
  float p[32];
  const int64_t lmax = a.L - 1;
  if constexpr (VPL == 2) {
    float2 x[32], z[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t l = min(l0 + j, lmax), l2 = max(l0 + j - shift, (int64_t)0);
      x[j] = __ldg(reinterpret_cast<const float2*>(V + l * MS) + lane);
      z[j] = __ldg(reinterpret_cast<const float2*>(V + l2 * MS) + lane);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float m2 = (l0 + j - shift >= 0) ? 1.f : 0.f;
      p[j] = fmaf(cw[0], x[j].x, cw[1] * x[j].y) + m2 * fmaf(ww[0], z[j].x, ww[1] * z[j].y);
    }
  } else {
    float x[32], z[32];
    const int ln = lane < ACT ? lane : 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t l = min(l0 + j, lmax), l2 = max(l0 + j - shift, (int64_t)0);
      x[j] = __ldg(V + l * MS + ln);
      z[j] = __ldg(V + l2 * MS + ln);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float m2 = (l0 + j - shift >= 0) ? 1.f : 0.f;
      p[j] = cw[0] * x[j] + m2 * (ww[0] * z[j]);
    }
  }
#pragma unroll
  for (int k = 16; k >= 1; k >>= 1) {
    const bool up = lane & k;
#pragma unroll
    for (int i = 0; i < k; ++i) {
      const float send = up ? p[i] : p[i + k];
      const float keep = up ? p[i + k] : p[i];
      p[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
    }
  }
  const int64_t l = l0 + lane;
  if (l < a.L) a.y[seq * a.L + l] = fmaf(dc, a.u[seq * a.L + l], p[0]);
}

// ============================================================================ fused derived data
// One CTA per channel: Krylov columns Kr[:, j] = Abar^j Bbar (j < 2^Kc) by doubling with the
// powers (Kr_{2^i + j} = P_i Kr_j, float64 FMA in ascending k as dgemm_batched_kernel), their
// tf32 hi/lo transpose krT, w = C P_Ne, and fp32 copies of C and D -- one launch instead of ~12.
__global__ void __launch_bounds__(256) bank_derived_kernel(const double* p64, int slots, const double* Bbar,
                                                           const double* C, const double* D, const int* Neff,
                                                           const int* Kc, double* Kr64, float* krT, double* w64,
                                                           float* w32, float* c32, float* d32, float* pvec,
                                                           int* tri, int fold, int ms, __half* kr16, float* kinv) {
  extern __shared__ double dsm[];
  double* Ps = dsm;                         // [ms][ms+1]
  double* Kr = Ps + ms * (ms + 1);          // [ms][129]
  const int s = blockIdx.x, tid = threadIdx.x;
  const int64_t mm = (int64_t)ms * ms;
  const int kc = Kc[s];
  const double* Ps0 = p64 + (int64_t)s * slots * mm;
  // NEXT-3: is Abar (slot 0) lower triangular? Then so are all its powers and the pair weights
  // (every upper entry of a product of lower-triangular matrices is a sum of products with a zero
  // factor: exactly 0), and the stage kernel skips their zero upper blocks.
  {
    int upper = 0;
    for (int e = tid; e < ms * ms; e += 256) upper |= (e % ms > e / ms) && Ps0[e] != 0.0;
    upper = __syncthreads_or(upper);
    if (tid == 0 && tri) tri[s] = upper ? 0 : 1;
  }
  for (int e = tid; e < ms * 128; e += 256) Kr[(e / 128) * 129 + e % 128] = (e % 128 == 0) ? Bbar[(int64_t)s * ms + e / 128] : 0.0;
  for (int i = 0; i < kc; ++i) {
    __syncthreads();
    for (int e = tid; e < ms * ms; e += 256) Ps[(e / ms) * (ms + 1) + e % ms] = Ps0[i * mm + e];
    __syncthreads();
    const int cols = 1 << i;
    if (ms == 64 && cols >= 8) {
      // Kr[:, cols + j] = P_i Kr[:, j] on the fp64 tensor path (mma.sync m8n8k4 f64): warp w owns
      // rows 8w..8w+7 and cols / 8 column tiles, K = 64 in 16 steps of 4
      const int w = tid / 32, lane = tid % 32, g = lane >> 2, t4 = lane & 3;
      for (int n0 = 0; n0 < cols; n0 += 64) {       // up to 8 column tiles per pass
        double d[8][2];
#pragma unroll
        for (int n = 0; n < 8; ++n) d[n][0] = d[n][1] = 0.0;
        const int ntile = (cols - n0) / 8 < 8 ? (cols - n0) / 8 : 8;
        for (int ks = 0; ks < 16; ++ks) {
          const double av = Ps[(8 * w + g) * (ms + 1) + 4 * ks + t4];
#pragma unroll
          for (int n = 0; n < 8; ++n) {
            if (n < ntile) {
              const double bv = Kr[(4 * ks + t4) * 129 + n0 + 8 * n + g];
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                           : "+d"(d[n][0]), "+d"(d[n][1]) : "d"(av), "d"(bv));
            }
          }
        }
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          if (n < ntile) {
            Kr[(8 * w + g) * 129 + cols + n0 + 8 * n + 2 * t4] = d[n][0];
            Kr[(8 * w + g) * 129 + cols + n0 + 8 * n + 2 * t4 + 1] = d[n][1];
          }
        }
      }
      continue;
    }
    for (int e = tid; e < ms * cols; e += 256) {   // Kr[r][cols + j] = sum_k P_i[r][k] Kr[k][j]
      const int r = e / cols, j = e % cols;
      double acc = 0.0;
      for (int k = 0; k < ms; ++k) acc = fma(Ps[r * (ms + 1) + k], Kr[k * 129 + j], acc);
      Kr[r * 129 + cols + j] = acc;
    }
  }
  __syncthreads();
  for (int e = tid; e < ms * 128; e += 256) {
    const int r = e / 128, j = e % 128;
    const double v = (j < (1 << kc)) ? Kr[r * 129 + j] : 0.0;
    Kr64[((int64_t)s * ms + r) * 128 + j] = v;
    const int kp = 127 - j;                        // krT[s][hi|lo][r][k'], k' = 127 - lag
    const float hi = tf32_rna((float)v);
    krT[(int64_t)s * 2 * ms * 128 + r * 128 + kp] = hi;
    krT[(int64_t)s * 2 * ms * 128 + ms * 128 + r * 128 + kp] = tf32_rna((float)(v - (double)hi));
  }
  // m = 64: the head's fp16 weights (R33) from the same Kr in shared memory: per column n
  // the exponent e_n of max_j |W_nj|, fp16 hi / lo of W * 2^(14 - e_n) at k' = 127 - j in the head's
  // shared-memory layout ([K chunk of 8][hi 64 | lo 64 rows][8]), and 2^(e_n - 14)
  if (kr16 != nullptr && ms == 64) {
    const int warp = tid / 32, lane = tid % 32;
    __half* Bh = kr16 + (int64_t)s * 2 * 128 * 64;
    for (int n = warp; n < 64; n += 8) {
      double x[4], mx = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = lane + 32 * q;
        x[q] = (j < (1 << kc)) ? Kr[n * 129 + j] : 0.0;
        mx = fmax(mx, fabs(x[q]));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const int e = mx > 0.0 ? max(-110, min(110, ilogb(mx))) : 0;
      if (lane == 0) kinv[(int64_t)s * 64 + n] = ldexpf(1.f, e - 14);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int kp = 127 - (lane + 32 * q), ch = kp / 8, o = kp % 8;
        const double xs = ldexp(x[q], 14 - e);
        const __half h = __double2half(xs);
        Bh[(ch * 128 + n) * 8 + o] = h;
        Bh[(ch * 128 + 64 + n) * 8 + o] = __double2half(xs - (double)__half2float(h));
      }
    }
  }
  // w = C P_Ne (row vector times matrix), and fp32 copies; P_Ne staged through shared memory
  const double* PN = Ps0 + (int64_t)Neff[s] * mm;
  __syncthreads();                                 // Ps (the last P_i) and Kr reads done
  for (int e = tid; e < ms * ms; e += 256) Ps[(e / ms) * (ms + 1) + e % ms] = PN[e];
  __syncthreads();
  for (int j = tid; j < ms; j += 256) {
    double acc = 0.0;
    for (int k = 0; k < ms; ++k) acc = fma(C[(int64_t)s * ms + k], Ps[k * (ms + 1) + j], acc);
    w64[(int64_t)s * ms + j] = acc;
    w32[(int64_t)s * ms + j] = (float)acc;
    c32[(int64_t)s * ms + j] = (float)C[(int64_t)s * ms + j];
  }
  if (tid == 0) d32[s] = D ? (float)D[s] : 0.f;
  // output-part row vectors (common.cuh OutParts): v_b = C prod_{i in b} P_{j0+i}, j0 = Ne - d, built
  // in float64 by multiplying in one stage at a time (the P's are powers of Abar and commute)
  if (pvec) {
    const int ne = Neff[s], d = fold_depth(ne, Kc[s], fold), j0 = ne - d;
    double* vs = Kr;                               // [kMaxParts][ms] float64 vectors (Kr no longer read)
    __syncthreads();
    for (int j = tid; j < ms; j += 256) vs[j] = C[(int64_t)s * ms + j];
    for (int q = 0; q <= d; ++q) {                 // vectors with bit q set from those without
      const double* Pq = Ps0 + (int64_t)(j0 + q) * mm;
      __syncthreads();
      for (int e = tid; e < ms * ms; e += 256) Ps[(e / ms) * (ms + 1) + e % ms] = Pq[e];
      __syncthreads();
      for (int e = tid; e < (1 << q) * ms; e += 256) {
        const int b = e / ms, j = e % ms;
        double acc = 0.0;
        for (int k = 0; k < ms; ++k) acc = fma(vs[b * ms + k], Ps[k * (ms + 1) + j], acc);
        vs[(b | (1 << q)) * ms + j] = acc;
      }
    }
    __syncthreads();
    for (int e = tid; e < (2 << d) * ms; e += 256) pvec[(int64_t)s * kMaxParts * ms + e] = (float)vs[e];
  }
}

int launch_bank_derived(const double* p64, int slots, const double* Bbar, const double* C, const double* D,
                        const int* Neff, const int* Kc, double* Kr64, float* krT, double* w64, float* w32,
                        float* c32, float* d32, float* pvec, int* tri, int fold, int n, int ms, cudaStream_t st,
                        void* kr16, float* kinv) {
  const size_t smem = (size_t)(ms * (ms + 1) + ms * 129) * sizeof(double);
  if (cudaFuncSetAttribute(bank_derived_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return CASC_ERR_CUDA;
  bank_derived_kernel<<<n, 256, smem, st>>>(p64, slots, Bbar, C, D, Neff, Kc, Kr64, krT, w64, w32, c32, d32, pvec,
                                            tri, fold, ms, static_cast<__half*>(kr16), kinv);
  CASC_LAUNCHED();
  return CASC_OK;
}

// ============================================================================ fused-output tail
// y_l = a_l + b_{l - 2^Ne} + d u_l with (a, b) = (C v, C P_Ne v) of the last state, written by
// the stage (or head) that produced v^(Ne): stage Ne and y = C v + D u in
// the regrouped form of R21/R24, without storing or re-reading v^(Ne).
__device__ __forceinline__ float4 f4add(float4 x, float4 y) { return make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w); }
// One (channel, sequence) per blockIdx.y, time rows along x; 4 rows per thread when every row
// offset is a multiple of 4 (L, the plane stride, the part shift h), so a shifted part is either
// wholly inside or wholly before the sequence for the 4 rows.
__global__ void bank_ab_tail_kernel(BankAbTailArg a) {
  const int64_t nseq = (a.list ? (int64_t)a.n_list : (int64_t)a.n_ch) * a.batch;
  const int64_t P = a.op.plane;
  const bool vec = (a.L % 4 == 0) && (P % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(a.u) | reinterpret_cast<uintptr_t>(a.y) |
                     reinterpret_cast<uintptr_t>(a.op.planes)) % 16 == 0);
  for (int64_t sq = blockIdx.y; sq < nseq; sq += gridDim.y) {
    const int ci = (int)(sq / a.batch), b = (int)(sq % a.batch);
    const int c = a.list ? a.list[ci] : ci;
    const int64_t base = ((int64_t)c * a.batch + b) * a.L;
    const int ne = a.op.neff[c];
    const int d = fold_depth(ne, a.op.kc[c], a.op.fold);
    const int np = 2 << d;                         // parts: stages ne-d .. ne applied here, shifts k*h
    const int64_t h = (int64_t)1 << (ne - d);
    const float dc = a.d[c];
    const float* pl = a.op.planes + base;
    if (vec && h % 4 == 0) {
      for (int64_t l = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); l < a.L; l += 4 * (int64_t)gridDim.x * blockDim.x) {
        float4 s = __ldcs(reinterpret_cast<const float4*>(pl + l));
        for (int k = 1; k < np; ++k)
          if (l >= k * h) s = f4add(s, __ldcs(reinterpret_cast<const float4*>(pl + k * P + l - k * h)));
        const float4 u4 = __ldcs(reinterpret_cast<const float4*>(a.u + base + l));
        __stcs(reinterpret_cast<float4*>(a.y + base + l),
               make_float4(fmaf(dc, u4.x, s.x), fmaf(dc, u4.y, s.y), fmaf(dc, u4.z, s.z), fmaf(dc, u4.w, s.w)));
      }
    } else {
      for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < a.L; l += (int64_t)gridDim.x * blockDim.x) {
        float s = pl[l];
        for (int k = 1; k < np; ++k)
          if (l >= k * h) s += pl[k * P + l - k * h];
        a.y[base + l] = fmaf(dc, a.u[base + l], s);
      }
    }
  }
}
int launch_bank_ab_tail(const BankAbTailArg& a, cudaStream_t st) {
  const int64_t nseq = (a.list ? (int64_t)a.n_list : (int64_t)a.n_ch) * a.batch;
  if (nseq <= 0 || a.L <= 0) return CASC_OK;
  const int64_t per_block = (a.L % 4 == 0 && a.op.plane % 4 == 0) ? 4 * 256 : 256;
  dim3 grid((unsigned)std::min<int64_t>(ceil_div(a.L, per_block), 64), (unsigned)std::min<int64_t>(nseq, 65535));
  bank_ab_tail_kernel<<<grid, 256, 0, st>>>(a);
  CASC_LAUNCHED();
  return CASC_OK;
}

// ============================================================================ launchers
template <int MS>
static int head_launch(const BankHeadArg& a, cudaStream_t st) {
  const size_t smem = (size_t)(2 * 128 * MS + 2 * 2 * 256 * 4 + 4 * 32 * MS) * sizeof(float);
  cudaFuncSetAttribute(bank_head_kernel<MS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t ntiles = ceil_div(a.L, 128);
  dim3 grid((unsigned)ceil_div(ntiles, a.tiles_per_cta), (unsigned)(a.n_list * a.batch));
  bank_head_kernel<MS><<<grid, 128, smem, st>>>(a);
  CASC_LAUNCHED();
  return CASC_OK;
}
template <int MS>
static int tail_launch(const BankTailArg& a, cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(a.L, 256), (unsigned)(a.n_ch * a.batch));
  bank_tail_kernel<MS><<<grid, 256, 0, st>>>(a);
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
