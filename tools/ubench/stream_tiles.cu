// Microbenchmark (diagnostics, not part of the library): HBM streaming with the access structure of
// the bank stage-pair pass (bank_hist.cu) and no arithmetic -- 148 CTAs, 32 KB tiles (128 rows x 64
// fp32) TMA-loaded into a ring of NS shared-memory slots by one producer warp, drained by four warps
// that write each 256-byte row back (a) with per-thread 256-bit global stores, as the pass does, or
// (b) in place in the slot + one TMA store per tile; (c) a plain float4 grid-stride copy for reference.
// Reports GB/s of read + write bytes.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/ubench/stream_tiles.cu -lcuda -o stream_tiles
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../../paper_2411_17729_b200/csrc/sm100.cuh"
using namespace casc::sm100;

constexpr int ROWS = 128, COLS = 64;
constexpr uint32_t CHUNK = ROWS * 128, SLOT = 2 * CHUNK;

__device__ __forceinline__ void tma_load2(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma_store2(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];"
               ::"l"(map), "r"(smem_u32(src)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void st8(float* p, const uint32_t* v) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]),
               "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
}

// position -> tile in the bank pass's residue-class order: sequences of 128 tiles, within one the
// chains r, r + S, r + 2S, ... (S = 1: the natural order)
__device__ __forceinline__ int chain_tile(int p, int S) {
  const int seq = p / 128, q = p % 128, J = 128 / S;
  return seq * 128 + (q / J) + (q % J) * S;
}
template <int NS, bool TMA_STORE>
__global__ void __launch_bounds__(160, 1) stream_kernel(const __grid_constant__ CUtensorMap src,
                                                        const __grid_constant__ CUtensorMap dstm, float* dst,
                                                        int ntiles, int S) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[NS], slot_free[NS];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&slot_free[s], 128); }
    fence_mbar_init();
  }
  __syncthreads();
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per, t1 = min(ntiles, t0 + per);
  if (warp == 0) {
    for (int t = t0, x = 0; t < t1; ++t, ++x) {
      const int s = x % NS;
      if (x >= NS) mbar_wait(&slot_free[s], (uint32_t)((x / NS - 1) & 1));
      if (lane == 0) {
        mbar_arrive_expect_tx(&full[s], SLOT);
        tma_load2(smem + s * SLOT, &src, &full[s], 0, chain_tile(t, S) * ROWS);
        tma_load2(smem + s * SLOT + CHUNK, &src, &full[s], 32, chain_tile(t, S) * ROWS);
      }
      __syncwarp();
    }
  } else {
    const int row = (warp - 1) * 32 + lane;
    for (int t = t0, x = 0; t < t1; ++t, ++x) {
      const int s = x % NS;
      mbar_wait(&full[s], (uint32_t)((x / NS) & 1));
      uint32_t v[64];
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) {
        const uint8_t* rr = smem + s * SLOT + kc * CHUNK + row * 128;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const float4 f = *reinterpret_cast<const float4*>(rr + ((cc ^ (row & 7)) * 16));
          const int o = kc * 32 + 4 * cc;
          v[o] = __float_as_uint(f.x + 1.f); v[o + 1] = __float_as_uint(f.y + 1.f);
          v[o + 2] = __float_as_uint(f.z + 1.f); v[o + 3] = __float_as_uint(f.w + 1.f);
        }
      }
      if constexpr (!TMA_STORE) {
        mbar_arrive(&slot_free[s]);
        float* orow = dst + ((int64_t)chain_tile(t, S) * ROWS + row) * COLS;
#pragma unroll
        for (int e = 0; e < 8; ++e) st8(orow + 8 * e, v + 8 * e);
      } else {
#pragma unroll
        for (int kc = 0; kc < 2; ++kc) {
          uint8_t* rr = smem + s * SLOT + kc * CHUNK + row * 128;
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) {
            const int o = kc * 32 + 4 * cc;
            *reinterpret_cast<float4*>(rr + ((cc ^ (row & 7)) * 16)) =
                make_float4(__uint_as_float(v[o]), __uint_as_float(v[o + 1]), __uint_as_float(v[o + 2]), __uint_as_float(v[o + 3]));
          }
        }
        fence_async_smem();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (row == 0) {
          tma_store2(&dstm, smem + s * SLOT, 0, chain_tile(t, S) * ROWS);
          tma_store2(&dstm, smem + s * SLOT + CHUNK, 32, chain_tile(t, S) * ROWS);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        mbar_arrive(&slot_free[s]);
      }
    }
  }
}

__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float4 f = a[i];
    f.x += 1.f;
    b[i] = f;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}
static void map2d(CUtensorMap* m, void* base, int64_t rows) {
  cuuint64_t dims[2] = {(cuuint64_t)COLS, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)COLS * 4};
  cuuint32_t box[2] = {32, ROWS}, es[2] = {1, 1};
  encode()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

template <class F>
static double time_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float t; cudaEventElapsedTime(&t, a, b);
    if (t < best) best = t;
  }
  return best;
}

int main() {
  const int ntiles = 96 * 1024;                         // 3 GiB per buffer
  const int64_t n = (int64_t)ntiles * ROWS * COLS;
  float *src, *dst;
  cudaMalloc(&src, n * 4); cudaMalloc(&dst, n * 4);
  cudaMemset(src, 0, n * 4);
  CUtensorMap ms, md;
  map2d(&ms, src, (int64_t)ntiles * ROWS);
  map2d(&md, dst, (int64_t)ntiles * ROWS);
  const double gb = 2.0 * n * 4 / 1e9;
  auto run = [&](auto kern, int ns, const char* name, int S) {
    const size_t smem = 1024 + (size_t)ns * SLOT;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const double ms_ = time_ms([&] { kern<<<148, 160, smem>>>(ms, md, dst, ntiles, S); });
    printf("%-28s slots %d S %3d: %.3f ms  %.0f GB/s  (%s)\n", name, ns, S, ms_, gb / ms_ * 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  for (int S : {1, 4, 16, 64}) {      // residue-class chain order of the bank pass (S = shift in tiles)
    run(stream_kernel<4, false>, 4, "tma load + st.global.v8", S);
    run(stream_kernel<4, true>, 4, "tma load + tma store", S);
  }
  const double mc = time_ms([&] { copy_kernel<<<148 * 8, 256>>>((const float4*)src, (float4*)dst, n / 4); });
  printf("%-28s        : %.3f ms  %.0f GB/s\n", "float4 copy", mc, gb / mc * 1e3);
  return 0;
}
