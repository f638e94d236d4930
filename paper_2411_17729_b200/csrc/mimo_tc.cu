// MIMO cascade stages on the sm_100a tensor cores (bf16 storage, fp32 accumulation).
//
// One kernel computes every step of PAPER.md:185-229 for a single system as a shifted
// multi-source GEMM with a fused residual epilogue:
//   out[b][l][n] = sum_src sum_k A_src[b][l - shift_src][k] W_src[n][k]  (+ R[b][l][n])
//   first stage  (a2): (u, 0, Bbar), (u, 1, Abar Bbar)            -> v^(1)
//   stage k      (a4): (v, 2^k, Abar^(2^k)) + residual v           -> v^(k+1)
//   last stage   (a5): (v, 0, C), (v, 2^N, C Abar^(2^N)), (u, 0, D) -> y
// The time shift is a TMA coordinate offset; rows l - shift < 0 fall outside the tensor and
// TMA zero-fills them, which is exactly "columns l < 2^k are left unchanged".
//
// Persistent CTAs (one per SM), 6 warps:
//   warp 0      TMA producer: 4-stage ring of {A 128x64, W BNx64} bf16 tiles (SWIZZLE_128B)
//   warp 1      MMA issuer: tcgen05.mma kind::f16, M=128, N=BN, K=16, into one of two TMEM
//               accumulators (2 x BN columns), commit -> smem slot free / accumulator full
//   warps 2-5   epilogue: TMEM -> registers (lane = time row), + residual tile (TMA-loaded,
//               SW128), convert to bf16 in place, TMA store; accumulator released to warp 1.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"
#include "mimo_tc.cuh"

namespace casc {
using namespace sm100;

namespace {
constexpr int BM = 128, BK = 64, STAGES = 4;
constexpr uint32_t A_BYTES = BM * BK * 2;          // 16 KB

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];"
               ::"l"(map), "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void prefetch_map(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(m) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_bf16(uint32_t u) {
  __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&u);
  return __bfloat1622float2(h);
}
}  // namespace

template <int BN>
__global__ void __launch_bounds__(192, 1) mimo_gemm_bf16_kernel(const __grid_constant__ MimoMaps maps, MimoArg a) {
  constexpr uint32_t B_BYTES = BN * BK * 2;
  constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr int TCOLS = 2 * BN < 32 ? 32 : 2 * BN;
  constexpr uint32_t R_BYTES = BM * 64 * 2;       // 16 KB epilogue chunk (128 rows x 64 cols)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                              // [STAGES][A_BYTES]
  uint8_t* sB = smem + STAGES * A_BYTES;           // [STAGES][B_BYTES]
  uint8_t* sR = sB + STAGES * B_BYTES;             // [2][R_BYTES]
  __shared__ uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2], rfull[2];
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t mt_per_b = (a.L + BM - 1) / BM;
  const int64_t n_mblk = mt_per_b * a.batch;
  const int n_nblk = (a.n_out + BN - 1) / BN;
  const int64_t n_tiles = n_mblk * n_nblk;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 128); mbar_init(&rfull[s], 1); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<TCOLS>(&tmem_base);
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < a.n_src; ++s) { prefetch_map(&maps.A[s]); prefetch_map(&maps.W[s]); }
    prefetch_map(&maps.out);
    if (a.has_residual) prefetch_map(&maps.R);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;

  if (warp == 0) {
    // =========================================================== TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t mb = tile / n_nblk;
        const int nb = (int)(tile % n_nblk);
        const int b = (int)(mb / mt_per_b);
        const int l0 = (int)((mb % mt_per_b) * BM);
        for (int src = 0; src < a.n_src; ++src) {
          const int nk = a.K[src] / BK;
          for (int kc = 0; kc < nk; ++kc) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
            tma_load_3d(sA + s * A_BYTES, &maps.A[src], &full[s], kc * BK, l0 - (int)a.shift[src], b);
            tma_load_2d(sB + s * B_BYTES, &maps.W[src], &full[s], kc * BK, nb * BN);
            if (++s == STAGES) { s = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // =========================================================== MMA issuer
    if (lane == 0) {
      const uint32_t idesc = make_idesc(FMT_BF16, BM, BN);
      int s = 0;
      uint32_t ph = 0;
      int64_t t_local = 0;
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t_local) {
        const int acc = (int)(t_local & 1);
        const uint32_t aph = (uint32_t)((t_local >> 1) & 1);
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tbase + acc * BN;
        bool first = true;
        for (int src = 0; src < a.n_src; ++src) {
          const int nk = a.K[src] / BK;
          for (int kc = 0; kc < nk; ++kc) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t a0 = smem_u32(sA + s * A_BYTES), b0 = smem_u32(sB + s * B_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t ad = make_sdesc(a0 + k * 32, 16, 1024, LAYOUT_SW128);
              const uint64_t bd = make_sdesc(b0 + k * 32, 16, 1024, LAYOUT_SW128);
              mma_f16(d, ad, bd, idesc, first ? 0u : 1u);
              first = false;
            }
            mma_commit(&empty[s]);
            if (++s == STAGES) { s = 0; ph ^= 1; }
          }
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else {
    // =========================================================== epilogue (warps 2..5)
    const int q = warp & 3;                       // TMEM lane quadrant of this warp
    const int row = q * 32 + lane;                // tile row = TMEM lane
    const bool leader = (warp == 2 && lane == 0);
    int64_t t_local = 0;
    uint32_t chunk_ctr = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t_local) {
      const int64_t mb = tile / n_nblk;
      const int nb = (int)(tile % n_nblk);
      const int b = (int)(mb / mt_per_b);
      const int l0 = (int)((mb % mt_per_b) * BM);
      const int acc = (int)(t_local & 1);
      mbar_wait(&tfull[acc], (uint32_t)((t_local >> 1) & 1));
      tc_fence_after();
      for (int j = 0; j < BN / 64; ++j, ++chunk_ctr) {
        const int rb = (int)(chunk_ctr & 1);
        uint8_t* rbuf = sR + rb * R_BYTES;
        const int n0 = nb * BN + j * 64;
        if (leader) {
          bulk_wait_read<1>();                     // the store that last used rbuf[rb] has read it
          if (a.has_residual) {
            mbar_arrive_expect_tx(&rfull[rb], R_BYTES);
            tma_load_3d(rbuf, &maps.R, &rfull[rb], n0, l0, b);
          }
        }
        uint32_t v[64];
        const uint32_t taddr = tbase + ((uint32_t)(q * 32) << 16) + acc * BN + j * 64;
        tmem_ld32(taddr, v);
        tmem_ld32(taddr + 32, v + 32);
        tmem_wait_ld();
        if (a.has_residual) mbar_wait(&rfull[rb], (chunk_ctr >> 1) & 1);
        else named_sync(2, 128);                   // rbuf free (leader waited for the old store)
        // row `row` of the SW128 tile: 8 chunks of 16 B at ((c ^ (row % 8)) * 16)
        uint8_t* rrow = rbuf + row * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint4* p = reinterpret_cast<uint4*>(rrow + ((c ^ (row & 7)) * 16));
          float f[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(v[c * 8 + e]);
          if (a.has_residual) {
            const uint4 r = *p;
            const float2 r0 = unpack_bf16(r.x), r1 = unpack_bf16(r.y), r2 = unpack_bf16(r.z), r3 = unpack_bf16(r.w);
            f[0] += r0.x; f[1] += r0.y; f[2] += r1.x; f[3] += r1.y;
            f[4] += r2.x; f[5] += r2.y; f[6] += r3.x; f[7] += r3.y;
          }
          *p = make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
        }
        fence_async_smem();
        named_sync(1, 128);
        if (leader) {
          tma_store_3d(&maps.out, rbuf, n0, l0, b);
          bulk_commit();
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
    if (leader) bulk_wait<0>();
  }
  __syncthreads();
  if (warp == 1) tmem_dealloc<TCOLS>(tbase);
}

// ----------------------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D bf16 signal [batch][L][K], box {64, rows, 1}, SWIZZLE_128B
static bool map_signal(CUtensorMap* m, const void* base, int64_t K, int64_t L, int64_t batch, int rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)L, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)(K * 2), (cuuint64_t)(L * K * 2)};
  cuuint32_t box[3] = {64, (cuuint32_t)rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// 2-D bf16 weight [n_out][K], box {64, BN}, SWIZZLE_128B
static bool map_weight(CUtensorMap* m, const void* base, int64_t K, int64_t n_out, int bn) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)n_out};
  cuuint64_t strides[1] = {(cuuint64_t)(K * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)bn};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool mimo_tc_supported(int m, int p, int q) {
  return m % 64 == 0 && p % 64 == 0 && q % 64 == 0 && m >= 64;
}

template <int BN>
static int launch_bn(const MimoGemm& g, cudaStream_t st) {
  MimoMaps maps;
  memset(&maps, 0, sizeof(maps));
  MimoArg a{};
  a.n_src = g.n_src;
  a.L = g.L;
  a.batch = g.batch;
  a.n_out = g.n_out;
  for (int s = 0; s < g.n_src; ++s) {
    if (g.src[s].K % BK) return CASC_ERR_UNSUPPORTED;
    a.K[s] = g.src[s].K;
    a.shift[s] = g.src[s].shift;
    if (!map_signal(&maps.A[s], g.src[s].A, g.src[s].K, g.L, g.batch, BM)) return CASC_ERR_CUDA;
    if (!map_weight(&maps.W[s], g.src[s].W, g.src[s].K, g.n_out, BN)) return CASC_ERR_CUDA;
  }
  a.has_residual = g.R != nullptr;
  if (g.R && !map_signal(&maps.R, g.R, g.n_out, g.L, g.batch, BM)) return CASC_ERR_CUDA;
  if (!map_signal(&maps.out, g.out, g.n_out, g.L, g.batch, BM)) return CASC_ERR_CUDA;
  const size_t smem = 1024 + STAGES * (A_BYTES + (size_t)BN * BK * 2) + 2 * BM * 64 * 2;
  if (cudaFuncSetAttribute(mimo_gemm_bf16_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return CASC_ERR_CUDA;
  const int64_t tiles = ceil_div(g.L, BM) * g.batch * ceil_div(g.n_out, BN);
  const int grid = (int)std::min<int64_t>(tiles, 148);
  mimo_gemm_bf16_kernel<BN><<<grid, 192, smem, st>>>(maps, a);
  CASC_LAUNCHED();
  return CASC_OK;
}

int launch_mimo_gemm_bf16(const MimoGemm& g, cudaStream_t st) {
  if (g.n_out % 256 == 0) return launch_bn<256>(g, st);
  if (g.n_out % 128 == 0) return launch_bn<128>(g, st);
  if (g.n_out % 64 == 0) return launch_bn<64>(g, st);
  return CASC_ERR_UNSUPPORTED;
}

}  // namespace casc
