// Batched float64 GEMM used for (a1) the repeated squaring P_{k+1} = P_k P_k of
// PAPER.md:164-166 and for the small derived products of the fused first / last stages
// (Abar Bbar, C P_N, C Bbar + D, C Abar Bbar). Powers are formed in float64 and rounded
// once afterwards, as PAPER.md:275-277 suggests ("powers ... can always be computed with a
// large number of accurate digits and used with as many digits as the application requires").
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace casc {

// 64x64 output tile per 256-thread block, 4x4 register micro-tile, K chunks of 16.
__global__ void __launch_bounds__(256) dgemm_batched_kernel(DgemmArg a) {
  const int s = blockIdx.z;
  if (a.skip_below && a.skip_below[s] < a.level) return;
  const int64_t selA = a.selA ? a.selA[s] : 0, selB = a.selB ? a.selB[s] : 0;
  const double* A = a.A + s * a.sA + selA * a.nA;
  const double* B = a.B + s * a.sB + selB * a.nB;
  double* C = a.C + s * a.sC;
  const double* Cadd = a.Cadd ? a.Cadd + s * a.sCadd : nullptr;

  __shared__ double As[16][64 + 1];
  __shared__ double Bs[16][64 + 1];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int row0 = blockIdx.y * 64, col0 = blockIdx.x * 64;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < a.K; k0 += 16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int e = tid + i * 256;             // 1024 elements of a 64x16 A chunk
      int r = e / 16, kk = e % 16;
      int gr = row0 + r, gk = k0 + kk;
      As[kk][r] = (gr < a.M && gk < a.K) ? A[(int64_t)gr * a.lda + gk] : 0.0;
      int kb = e / 64, c = e % 64;       // 16x64 B chunk
      int gkb = k0 + kb, gc = col0 + c;
      Bs[kb][c] = (gkb < a.K && gc < a.N) ? B[(int64_t)gkb * a.ldb + gc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int gr = row0 + ty * 4 + i;
    if (gr >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gc = col0 + tx * 4 + j;
      if (gc >= a.N) continue;
      double v = acc[i][j];
      if (Cadd) v += Cadd[(int64_t)gr * a.ldc + gc];
      C[(int64_t)gr * a.ldc + gc] = v;
    }
  }
}

// The same batched GEMM on the fp64 tensor path (mma.sync m8n8k4 f64, DMMA): 64 x 64 output tile
// per 256-thread CTA, warp w owns rows 8w..8w+7 (eight 8 x 8 column tiles), K in chunks of 32 staged
// through shared memory (zero-filled past M, N, K). Per element a float64 dot product of the same
// terms as dgemm_batched_kernel in another summation order (both are float64 FMA chains). The
// MIMO squarings (m = 256: E3, m = 1024: E4, 11 squarings of 2 m^3 flops per step) run here.
// One 64 x 64 output tile C[row0:, col0:] (+ Cadd) of C = A B on the fp64 tensor path (mma.sync
// m8n8k4 f64, DMMA) by a 256-thread CTA: warp w owns rows 8w..8w+7 (eight 8 x 8 column tiles); K in
// chunks of 16 staged through shared memory with cp.async double buffering (the next chunk's loads
// overlap this chunk's DMMAs; zero-filled past M, N, K).
constexpr int kDKC = 16;                                   // K chunk of the 32 x 32 tiles' loads
template <int KC>
struct Dmma64 {
  static constexpr int LA = KC + 4, LB = 72;               // padded strides (doubles)
  static constexpr size_t BYTES = sizeof(double) * 2 * (64 * LA + KC * LB);
};
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(valid ? src : nullptr), "r"(valid ? 8 : 0) : "memory");
}
template <int KC>
__device__ __forceinline__ void dmma_tile(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                                          int64_t ldc, const double* Cadd, int M, int N, int K, int row0, int col0,
                                          double* smem) {
  using D = Dmma64<KC>;
  double* sA[2] = {smem, smem + 64 * D::LA};
  double* sB[2] = {smem + 2 * 64 * D::LA, smem + 2 * 64 * D::LA + KC * D::LB};
  const int tid = threadIdx.x, w = tid / 32, lane = tid % 32, g = lane >> 2, t4 = lane & 3;
  auto load = [&](int buf, int k0) {
#pragma unroll
    for (int i = 0; i < 64 * KC / 256; ++i) {
      const int e = tid + i * 256;
      const int r = e / KC, kk = e % KC;                 // A chunk 64 x KC
      const int gr = row0 + r, gk = k0 + kk;
      const bool va = gr < M && gk < K;
      cp_async8(&sA[buf][r * D::LA + kk], A + (va ? (int64_t)gr * lda + gk : 0), va);
      const int kb = e / 64, c = e % 64;                 // B chunk KC x 64
      const int gkb = k0 + kb, gc = col0 + c;
      const bool vb = gkb < K && gc < N;
      cp_async8(&sB[buf][kb * D::LB + c], B + (vb ? (int64_t)gkb * ldb + gc : 0), vb);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double d[8][2];
#pragma unroll
  for (int n = 0; n < 8; ++n) d[n][0] = d[n][1] = 0.0;
  const int nch = (K + KC - 1) / KC;
  load(0, 0);
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    if (c + 1 < nch) {
      load(buf ^ 1, (c + 1) * KC);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) {
      const double av = sA[buf][(8 * w + g) * D::LA + 4 * ks + t4];
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        const double bv = sB[buf][(4 * ks + t4) * D::LB + 8 * n + g];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(d[n][0]), "+d"(d[n][1]) : "d"(av), "d"(bv));
      }
    }
    __syncthreads();                                     // buf is refilled by the next iteration's prefetch
  }
  const int gr = row0 + 8 * w + g;
  if (gr >= M) return;
#pragma unroll
  for (int n = 0; n < 8; ++n) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gc = col0 + 8 * n + 2 * t4 + h;
      if (gc >= N) continue;
      double v = d[n][h];
      if (Cadd) v += Cadd[(int64_t)gr * ldc + gc];
      C[(int64_t)gr * ldc + gc] = v;
    }
  }
}

// A 32 x 32 output tile of C = A B by a 256-thread CTA on the same DMMA path (the cooperative
// squarings at m <= 512: four times the tiles per level of the 64 x 64 form, e.g. 64 instead of 16 at
// m = 256, so the level's dependent chain is spread over more SMs). Warp w owns rows 8 (w % 4) ..
// +8 and columns 16 (w / 4) .. +16 (two 8 x 8 tiles); K in chunks of KC with cp.async double
// buffering (KC = 64: four L2 round trips per tile at K = 256 instead of sixteen). Each element is
// the same DMMA chain over K as in dmma_tile (same order): bitwise equal.
template <int KC>
struct Dmma32 {
  static constexpr int LA = KC + 4, LB = 36;     // padded strides (doubles): conflict-free fragment loads
  static constexpr size_t BYTES = sizeof(double) * 2 * (32 * LA + KC * LB);
};
template <int KC>
__device__ __forceinline__ void dmma_tile32(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                                            int64_t ldc, int M, int N, int K, int row0, int col0, double* smem) {
  using D = Dmma32<KC>;
  double* sA[2] = {smem, smem + 32 * D::LA};
  double* sB[2] = {smem + 2 * 32 * D::LA, smem + 2 * 32 * D::LA + KC * D::LB};
  const int tid = threadIdx.x, w = tid / 32, lane = tid % 32, g = lane >> 2, t4 = lane & 3;
  const int r0 = 8 * (w & 3), c0 = 16 * (w >> 2);
  auto load = [&](int buf, int k0) {
#pragma unroll
    for (int i = 0; i < 32 * KC / 256; ++i) {
      const int e = tid + i * 256;
      const int r = e / KC, kk = e % KC;                 // A chunk 32 x KC
      const int gr = row0 + r, gk = k0 + kk;
      const bool va = gr < M && gk < K;
      cp_async8(&sA[buf][r * D::LA + kk], A + (va ? (int64_t)gr * lda + gk : 0), va);
      const int kb = e / 32, c = e % 32;                 // B chunk KC x 32
      const int gkb = k0 + kb, gc = col0 + c;
      const bool vb = gkb < K && gc < N;
      cp_async8(&sB[buf][kb * D::LB + c], B + (vb ? (int64_t)gkb * ldb + gc : 0), vb);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  const int nch = (K + KC - 1) / KC;
  load(0, 0);
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    if (c + 1 < nch) {
      load(buf ^ 1, (c + 1) * KC);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) {
      const double av = sA[buf][(r0 + g) * D::LA + 4 * ks + t4];
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        const double bv = sB[buf][(4 * ks + t4) * D::LB + c0 + 8 * n + g];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(d[n][0]), "+d"(d[n][1]) : "d"(av), "d"(bv));
      }
    }
    __syncthreads();
  }
  const int gr = row0 + r0 + g;
  if (gr >= M) return;
#pragma unroll
  for (int n = 0; n < 2; ++n)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gc = col0 + c0 + 8 * n + 2 * t4 + h;
      if (gc < N) C[(int64_t)gr * ldc + gc] = d[n][h];
    }
}
constexpr int kPowKC = 64;

// The same batched GEMM on the fp64 tensor path: one 64 x 64 tile per CTA. Per element a float64
// dot product of the same terms as dgemm_batched_kernel in another summation order (both are
// float64 FMA chains).
// (32 WR) x (32 WC) output tile by WR x WC warps, each warp a 32 x 32 block (4 x 4 DMMA tiles: 8
// fragment loads per 16 DMMAs instead of 9 per 8), K chunks of 16 double-buffered. Same per-element
// DMMA chain over K as dmma_tile: bitwise equal.
template <int WR, int WC>
struct DmmaW32 {
  static constexpr int KC = 16, TR = 32 * WR, TC = 32 * WC, NT = 32 * WR * WC;
  static constexpr int LA = KC + 4, LB = TC == 32 ? 36 : 72;
  double A[2][TR * LA];
  double B[2][KC * LB];
};
template <int WR, int WC>
__device__ __forceinline__ void dmma_tile_w32(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                                              int64_t ldc, const double* Cadd, int M, int N, int K, int row0,
                                              int col0, DmmaW32<WR, WC>& sm) {
  using D = DmmaW32<WR, WC>;
  constexpr int KC = D::KC, TR = D::TR, TC = D::TC, NT = D::NT, LA = D::LA, LB = D::LB;
  auto& sA = sm.A;
  auto& sB = sm.B;
  const int tid = threadIdx.x, w = tid / 32, lane = tid % 32, g = lane >> 2, t4 = lane & 3;
  const int r0 = 32 * (w % WR), c0 = 32 * (w / WR);
  auto load = [&](int buf, int k0) {
#pragma unroll
    for (int i = 0; i < TR * KC / NT; ++i) {
      const int e = tid + i * NT;
      const int r = e / KC, kk = e % KC;
      const int gr = row0 + r, gk = k0 + kk;
      const bool va = gr < M && gk < K;
      cp_async8(&sA[buf][r * LA + kk], A + (va ? (int64_t)gr * lda + gk : 0), va);
    }
#pragma unroll
    for (int i = 0; i < TC * KC / NT; ++i) {
      const int e = tid + i * NT;
      const int kb = e / TC, c = e % TC;
      const int gkb = k0 + kb, gc = col0 + c;
      const bool vb = gkb < K && gc < N;
      cp_async8(&sB[buf][kb * LB + c], B + (vb ? (int64_t)gkb * ldb + gc : 0), vb);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double d[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) d[i][j][0] = d[i][j][1] = 0.0;
  const int nch = (K + KC - 1) / KC;
  load(0, 0);
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    if (c + 1 < nch) {
      load(buf ^ 1, (c + 1) * KC);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = sA[buf][(r0 + 8 * i + g) * LA + 4 * ks + t4];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = sB[buf][(4 * ks + t4) * LB + c0 + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(d[i][j][0]), "+d"(d[i][j][1]) : "d"(av[i]), "d"(bv[j]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gr = row0 + r0 + 8 * i + g;
    if (gr >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gc = col0 + c0 + 8 * j + 2 * t4 + h;
        if (gc >= N) continue;
        double v = d[i][j][h];
        if (Cadd) v += Cadd[(int64_t)gr * ldc + gc];
        C[(int64_t)gr * ldc + gc] = v;
      }
  }
}
template <int WR, int WC>
__global__ void __launch_bounds__(32 * WR * WC) dgemm_mma_w32_kernel(DgemmArg a) {
  __shared__ __align__(16) DmmaW32<WR, WC> sm;
  const int s = blockIdx.z;
  if (a.skip_below && a.skip_below[s] < a.level) return;
  const int64_t selA = a.selA ? a.selA[s] : 0, selB = a.selB ? a.selB[s] : 0;
  dmma_tile_w32<WR, WC>(a.A + s * a.sA + selA * a.nA, a.lda, a.B + s * a.sB + selB * a.nB, a.ldb, a.C + s * a.sC, a.ldc,
                        a.Cadd ? a.Cadd + s * a.sCadd : nullptr, a.M, a.N, a.K, blockIdx.y * DmmaW32<WR, WC>::TR,
                        blockIdx.x * DmmaW32<WR, WC>::TC, sm);
}

template <int KC>
__global__ void __launch_bounds__(256) dgemm_mma_kernel(DgemmArg a) {
  const int s = blockIdx.z;
  if (a.skip_below && a.skip_below[s] < a.level) return;
  const int64_t selA = a.selA ? a.selA[s] : 0, selB = a.selB ? a.selB[s] : 0;
  extern __shared__ __align__(16) double sm[];
  dmma_tile<KC>(a.A + s * a.sA + selA * a.nA, a.lda, a.B + s * a.sB + selB * a.nB, a.ldb, a.C + s * a.sC, a.ldc,
            a.Cadd ? a.Cadd + s * a.sCadd : nullptr, a.M, a.N, a.K, blockIdx.y * 64, blockIdx.x * 64, sm);
}

// a1 for one system with m > 64 (MIMO: E3 m = 256, E4 m = 1024) in ONE cooperative launch: P_0 =
// Abar, then N squarings P_k = P_{k-1} P_{k-1} (each level's 32 x 32 tiles spread over the resident
// CTAs, a grid-wide barrier between levels), then every P_k rounded once to its storage image (tf32
// hi/lo or bf16). Replaces N + 2 launches whose fixed latency dominated at m = 256 (16 tiles per
// level: 13 launches of ~29 us for 33 MFLOP each).
__global__ void __launch_bounds__(256, 2) powers_coop_kernel(const double* Abar, double* p64, float* f32,
                                                          __nv_bfloat16* b16, int N, int m) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  const int64_t mm = (int64_t)m * m;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gsz = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = gtid; e < mm; e += gsz) p64[e] = Abar[e];
  grid.sync();
  const int tn = (m + 31) / 32, tiles = tn * tn;
  for (int k = 1; k <= N; ++k) {
    const double* Pk = p64 + (k - 1) * mm;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x)
      dmma_tile32<kPowKC>(Pk, m, Pk, m, p64 + k * mm, m, m, m, m, (t / tn) * 32, (t % tn) * 32, sm);
    grid.sync();
  }
  for (int64_t e = gtid; e < (int64_t)(N + 1) * mm; e += gsz) {
    const int64_t slot = e / mm, ij = e % mm;
    const double p = p64[e];
    if (f32) {
      const float hi = tf32_rna((float)p);
      f32[slot * 2 * mm + ij] = hi;
      f32[slot * 2 * mm + mm + ij] = tf32_rna((float)(p - (double)hi));
    }
    if (b16) b16[e] = __float2bfloat16_rn((float)p);
  }
}

__global__ void __launch_bounds__(256, 2) derived_coop_kernel(const __grid_constant__ DerivedPlan pl) {
  cg::grid_group grid = cg::this_grid();
  __shared__ __align__(16) double sm[Dmma64<kDKC>::BYTES / sizeof(double)];
  for (int ph = 0; ph < 2; ++ph) {
    int base = 0;                                          // tiles of this phase's jobs, concatenated
    for (int j = 0; j < pl.n_jobs; ++j) {
      const DJob& J = pl.jobs[j];
      if (J.phase != ph) continue;
      const int tm = (J.M + 63) / 64, tn = (J.N + 63) / 64;
      for (int t = (int)blockIdx.x - base; t < tm * tn; t += gridDim.x)
        if (t >= 0) dmma_tile<kDKC>(J.A, J.lda, J.B, J.ldb, J.C, J.ldc, J.Cadd, J.M, J.N, J.K, (t / tn) * 64, (t % tn) * 64, sm);
      base = (base + tm * tn) % gridDim.x;                 // spread the next job's tiles onto other CTAs
    }
    grid.sync();
  }
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gsz = (int64_t)gridDim.x * blockDim.x;
  for (int c = 0; c < pl.n_convs; ++c) {
    const DConv& C = pl.convs[c];
    for (int64_t e = gtid; e < C.n; e += gsz) {
      const double x = C.src[e];
      if (pl.tf32) {
        float* d = static_cast<float*>(C.dst);
        const float hi = tf32_rna((float)x);
        d[e] = hi;
        d[C.n + e] = tf32_rna((float)(x - (double)hi));
      } else {
        static_cast<__nv_bfloat16*>(C.dst)[e] = __float2bfloat16_rn((float)x);
      }
    }
  }
}

int launch_derived_coop(const DerivedPlan& plan, cudaStream_t st) {
  int dev = 0, sms = 148, per_sm = 0;
  CASC_TRY(cudaGetDevice(&dev));
  CASC_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CASC_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, derived_coop_kernel, 256, 0));
  const int grid = sms * std::max(1, std::min(per_sm, 2));
  void* args[] = {(void*)&plan};
  CASC_TRY(cudaLaunchCooperativeKernel((const void*)derived_coop_kernel, dim3(grid), dim3(256), args, 0, st));
  CASC_LAUNCHED();
  return CASC_OK;
}

int launch_powers_coop(const PackLayout& P, const double* Abar, int N, int m, cudaStream_t st) {
  int dev = 0, sms = 148, per_sm = 0;
  CASC_TRY(cudaGetDevice(&dev));
  CASC_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t smem = Dmma32<kPowKC>::BYTES;
  CASC_TRY(cudaFuncSetAttribute(powers_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CASC_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, powers_coop_kernel, 256, smem));
  const int tn = (m + 31) / 32;
  int grid = std::min(sms * std::max(per_sm, 1), std::max(tn * tn, sms));
  double* p64 = P.p64;
  float* f32 = P.f32;
  __nv_bfloat16* b16 = P.b16;
  void* args[] = {(void*)&Abar, (void*)&p64, (void*)&f32, (void*)&b16, (void*)&N, (void*)&m};
  CASC_TRY(cudaLaunchCooperativeKernel((const void*)powers_coop_kernel, dim3(grid), dim3(256), args, smem, st));
  CASC_LAUNCHED();
  return CASC_OK;
}

int launch_dgemm(const DgemmArg& a, int n_sys, cudaStream_t st) {
  if (a.M <= 0 || a.N <= 0 || n_sys <= 0) return CASC_OK;
  dim3 grid((unsigned)ceil_div(a.N, 64), (unsigned)ceil_div(a.M, 64), (unsigned)n_sys);
  // the tensor path for full-width products; thin ones (a row vector times a matrix) on FMA. Long
  // contractions (E4's squarings, K = 1024) on 128-thread CTAs whose warps own 32 x 32 blocks:
  // 1.83 -> 1.65 ms per E4 step (A/B; 32 x 32 or 64 x 32 tiles, and K chunks of 32 or 64, slower)
  if (a.M >= 64 && a.N >= 64 && a.K >= 256) dgemm_mma_w32_kernel<2, 2><<<grid, 128, 0, st>>>(a);
  else if (a.M >= 32 && a.N >= 32) dgemm_mma_kernel<kDKC><<<grid, 256, Dmma64<kDKC>::BYTES, st>>>(a);
  else dgemm_batched_kernel<<<grid, 256, 0, st>>>(a);
  CASC_LAUNCHED();
  return CASC_OK;
}

// Round each float64 power once to the storage format (R17):
//   FP32 mode: hi = rna_tf32(fp32(P)), lo = rna_tf32(fp32(P - hi))  -> P ~ hi + lo to ~2^-22
//   BF16 mode: RN-even bf16 of fp32(P)
__global__ void pack_powers_kernel(const int* hdr, const double* p64, float* f32,
                                   __nv_bfloat16* b16, int n_sys, int N_max, int m) {
  const int64_t mm = (int64_t)m * m;
  const int64_t total = (int64_t)n_sys * (N_max + 1) * mm;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t slot = e / mm, ij = e % mm;
    const int s = (int)(slot / (N_max + 1)), k = (int)(slot % (N_max + 1));
    if (k > hdr[s]) continue;
    const double p = p64[e];
    if (f32) {
      float hi = tf32_rna((float)p);
      float lo = tf32_rna((float)(p - (double)hi));
      f32[slot * 2 * mm + ij] = hi;
      f32[slot * 2 * mm + mm + ij] = lo;
    }
    if (b16) b16[e] = __float2bfloat16_rn((float)p);
  }
}

int launch_pack(const PackLayout& P, int n_sys, int N_max, int m, cudaStream_t st) {
  const int64_t total = (int64_t)n_sys * (N_max + 1) * m * m;
  int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
  pack_powers_kernel<<<blocks, 256, 0, st>>>(P.hdr, P.p64, P.f32, P.b16, n_sys, N_max, m);
  CASC_LAUNCHED();
  return CASC_OK;
}

// a1 for small systems (m <= 64, the HiPPO banks): one CTA per system squares P_k in shared
// memory N_s times (float64 FMA in ascending k, the same order as dgemm_batched_kernel, so the
// powers are bitwise those of the per-level launches) and writes each P_k and its storage image
// as soon as it is formed -- one launch instead of N_max + 1.
__global__ void __launch_bounds__(256) powers_small_kernel(const double* Abar, const int* hdr, double* p64,
                                                           float* f32, __nv_bfloat16* b16, int N_max, int m) {
  // row stride 72 doubles: the B-fragment loads (lanes g = 0..7 along a row, t4 = 0..3 down four
  // rows) fall in two disjoint halves of the banks, 2 wavefronts per load (stride 65: 4)
  constexpr int LD = 72;
  __shared__ double S[64 * LD];                          // P_k; P_{k+1} overwrites it in place
  const int s = blockIdx.x, tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int64_t mm = (int64_t)m * m;
  const int Ns = hdr[s];
  const double* A0 = Abar + (int64_t)s * mm;
  for (int e = tid; e < m * m; e += 256) S[(e / m) * LD + e % m] = A0[e];
  __syncthreads();
  for (int k = 0; k <= Ns; ++k) {
    const double* Pk = S;
    const int64_t slot = (int64_t)s * (N_max + 1) + k;
    for (int e = tid; e < m * m; e += 256) {             // P_k out: float64 + storage image
      const double p = Pk[(e / m) * LD + e % m];
      p64[slot * mm + e] = p;
      if (f32) {
        const float hi = tf32_rna((float)p);
        f32[slot * 2 * mm + e] = hi;
        f32[slot * 2 * mm + mm + e] = tf32_rna((float)(p - (double)hi));
      }
      if (b16) b16[slot * mm + e] = __float2bfloat16_rn((float)p);
    }
    if (k == Ns) break;
    if (m == 64) {
      // P_{k+1} = P_k P_k on the fp64 tensor path (mma.sync m8n8k4 f64; per-element fused
      // multiply-adds in float64 like the FMA loop below, in a different summation order): warp w
      // owns rows 8w..8w+7, eight 8 x 8 column tiles, K = 64 in 16 steps of 4
      const int w = tid / 32, lane = tid % 32, g = lane >> 2, t4 = lane & 3;
      double d[8][2];
#pragma unroll
      for (int n = 0; n < 8; ++n) d[n][0] = d[n][1] = 0.0;
#pragma unroll 4
      for (int ks = 0; ks < 16; ++ks) {
        const double av = Pk[(8 * w + g) * LD + 4 * ks + t4];
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          const double bv = Pk[(4 * ks + t4) * LD + 8 * n + g];
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(d[n][0]), "+d"(d[n][1]) : "d"(av), "d"(bv));
        }
      }
      __syncthreads();                                  // all reads of P_k done
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        S[(8 * w + g) * LD + 8 * n + 2 * t4] = d[n][0];
        S[(8 * w + g) * LD + 8 * n + 2 * t4 + 1] = d[n][1];
      }
      __syncthreads();
      continue;
    }
    double acc[4][4] = {};                              // P_{k+1} = P_k P_k
    for (int kk = 0; kk < m; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = (ty * 4 + i < m) ? Pk[(ty * 4 + i) * LD + kk] : 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = (tx * 4 + j < m) ? Pk[kk * LD + tx * 4 + j] : 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();                                    // all reads of P_k done
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (ty * 4 + i < m && tx * 4 + j < m) S[(ty * 4 + i) * LD + tx * 4 + j] = acc[i][j];
    __syncthreads();
  }
}

int launch_powers_small(const PackLayout& P, const double* Abar, int n_sys, int N_max, int m, cudaStream_t st) {
  if (m > 64) return CASC_ERR_UNSUPPORTED;
  powers_small_kernel<<<n_sys, 256, 0, st>>>(Abar, P.hdr, P.p64, P.f32, P.b16, N_max, m);
  CASC_LAUNCHED();
  return CASC_OK;
}

// Diagnostics for the planner (casc_powers_norms): sums of squares of the stored float64 powers
// P_k (k <= N_s) of every system, and of the first neglected power P_{N_s+1} = P_{N_s} P_{N_s},
// formed 16 x 16 entries per block in registers (float64 FMA) and reduced, never stored.
// acc [n_sys][N_max + 2] (zeroed by the caller).
__global__ void powers_sumsq_kernel(const double* p64, const int* hdr, int N_max, int m, double* acc) {
  const int s = blockIdx.y, k = blockIdx.z;               // system, power index 0..N_max
  if (k > hdr[s]) return;
  const int64_t mm = (int64_t)m * m;
  const double* P = p64 + ((int64_t)s * (N_max + 1) + k) * mm;
  double t = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < mm; e += (int64_t)gridDim.x * blockDim.x)
    t = fma(P[e], P[e], t);
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(acc + (int64_t)s * (N_max + 2) + k, t);
}
__global__ void next_power_sumsq_kernel(const double* p64, const int* hdr, int N_max, int m, double* acc) {
  const int s = blockIdx.z, Ns = hdr[s];
  const int64_t mm = (int64_t)m * m;
  const double* P = p64 + ((int64_t)s * (N_max + 1) + Ns) * mm;
  __shared__ double As[16][17], Bs[16][17];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int row = blockIdx.y * 16 + ty, col = blockIdx.x * 16 + tx;
  double c = 0.0;
  for (int k0 = 0; k0 < m; k0 += 16) {
    As[ty][tx] = (row < m && k0 + tx < m) ? P[(int64_t)row * m + k0 + tx] : 0.0;
    Bs[ty][tx] = (k0 + ty < m && col < m) ? P[(int64_t)(k0 + ty) * m + col] : 0.0;
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) c = fma(As[ty][kk], Bs[kk][tx], c);
    __syncthreads();
  }
  double t = c * c;
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(acc + (int64_t)s * (N_max + 2) + Ns + 1, t);
}
int launch_powers_sumsq(const PackLayout& P, int n_sys, int N_max, int m, double* acc, cudaStream_t st) {
  const int64_t mm = (int64_t)m * m;
  dim3 g1((unsigned)std::min<int64_t>(ceil_div(mm, 256), 64), (unsigned)n_sys, (unsigned)(N_max + 1));
  powers_sumsq_kernel<<<g1, 256, 0, st>>>(P.p64, P.hdr, N_max, m, acc);
  CASC_LAUNCHED();
  dim3 g2((unsigned)ceil_div(m, 16), (unsigned)ceil_div(m, 16), (unsigned)n_sys);
  next_power_sumsq_kernel<<<g2, 256, 0, st>>>(P.p64, P.hdr, N_max, m, acc);
  CASC_LAUNCHED();
  return CASC_OK;
}

__global__ void f64_to_f32_kernel(const double* src, float* dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (float)src[i];
}

int launch_f64_to_f32(const double* src, float* dst, int64_t n, cudaStream_t st) {
  if (n <= 0) return CASC_OK;
  int blocks = (int)std::min<int64_t>(ceil_div(n, 256), 148 * 8);
  f64_to_f32_kernel<<<blocks, 256, 0, st>>>(src, dst, n);
  CASC_LAUNCHED();
  return CASC_OK;
}

}  // namespace casc
