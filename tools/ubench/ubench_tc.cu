// Microbenchmarks (diagnostics, not part of the library): TMEM load bandwidth, tcgen05.mma
// kind::tf32 issue rate with both operands in shared memory (SS) or A in TMEM (TS), and the
// shared-memory read bandwidth, on one SM. Build: nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2411_17729_b200/csrc/sm100.cuh"
using namespace casc::sm100;

__device__ __forceinline__ int lane_id() { return threadIdx.x % 32; }
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void ld128nw(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
      "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
        "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
        "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
}
// warp-collective issue: the whole (converged) warp executes this; one elected lane issues the MMA
__device__ __forceinline__ void mma_ss_w(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts_w(uint32_t d, uint32_t a, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(bd), "r"(idesc), "r"(acc));
}
__global__ void k_mma_w(int mode, int N, int iters, unsigned long long* out, int nacc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) {
    const uint32_t idesc = make_idesc(FMT_TF32, 128, N);
    const uint32_t a0 = smem_u32(sm), b0 = a0 + 16384;
    const uint64_t ad0 = make_sdesc(a0, 16, 1024, LAYOUT_SW128), bd0 = make_sdesc(b0, 16, 1024, LAYOUT_SW128);
    const uint32_t stride = (uint32_t)(N > 64 ? N : 64);
    const uint32_t t = tb;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t dd = t + (nacc == 1 ? 0u : (uint32_t)((k % nacc) * stride));
        if (mode == 0) mma_ss_w(dd, ad0 + 2 * k, bd0 + 2 * k, idesc, 1);
        else mma_ts_w(dd, t + 448 + k * 8, bd0 + 2 * k, idesc, 1);
      }
    }
    if (threadIdx.x == 0) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tb);
}

// nw warps issue concurrently, warp w into accumulator columns [w*128, w*128+N); TS: A in TMEM
template <bool TS>
__global__ void k_mma_mw(int N, int iters, unsigned long long* out, int nw) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ uint64_t bar[4];
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const int warp = threadIdx.x / 32;
  const long long t0 = clock64();
  if (warp < nw) {
    const uint32_t idesc = make_idesc(FMT_TF32, 128, N);
    const uint32_t a0 = smem_u32(sm), b0 = a0 + 16384;
    const uint64_t ad0 = make_sdesc(a0, 16, 1024, LAYOUT_SW128), bd0 = make_sdesc(b0, 16, 1024, LAYOUT_SW128);
    const uint32_t dd = tb + (uint32_t)(warp * 128);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (!TS) mma_ss_w(dd, ad0 + 2 * k, bd0 + 2 * k, idesc, 1);
        else mma_ts_w(dd, tb + 384 + k * 8, bd0 + 2 * k, idesc, 1);
      }
    }
    if (threadIdx.x % 32 == 0) mma_commit(&bar[warp]);
    __syncwarp();
    mbar_wait(&bar[warp], 0);
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tb);
}

// pattern of the 3xTF32 GEMM: per K-step mma(d, A_hi, W_hi), mma(dc, A_lo, W_hi), mma(dc, A_hi, W_lo)
// mode 0: d != dc (two accumulators), mode 1: d == dc (one accumulator); A in TMEM
template <int MODE>
__global__ void k_mma_3x(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const long long t0 = clock64();
  if (threadIdx.x < 32) {
    const uint32_t idesc = make_idesc(FMT_TF32, 128, 64);
    const uint64_t bd0 = make_sdesc(smem_u32(sm) + 16384, 16, 1024, LAYOUT_SW128);
    const uint32_t d = tb, dc = MODE == 0 ? tb + 64 : tb, ah = tb + 256, al = tb + 288;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        mma_ts_w(d, ah + k * 8, bd0 + 2 * k, idesc, 1);
        mma_ts_w(dc, al + k * 8, bd0 + 2 * k, idesc, 1);
        mma_ts_w(dc, ah + k * 8, bd0 + 512 + 2 * k, idesc, 1);
      }
    }
    if (threadIdx.x == 0) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tb);
}

// TMEM contention: warp 0 issues the 3xTF32 TS pattern (N = 64) while warps 2-5 load and/or
// warps 6-9 store TMEM (epilogue / transform traffic); cycles per MMA
__global__ void k_contend(int iters, int ld_on, int st_on, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); stop = 0; }
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const int warp = threadIdx.x / 32;
  float acc = 0.f;
  if (warp == 0) {
    const uint32_t idesc = make_idesc(FMT_TF32, 128, 64);
    const uint64_t bd0 = make_sdesc(smem_u32(sm) + 16384, 16, 1024, LAYOUT_SW128);
    const uint32_t d = tb, dc = tb + 64, ah = tb + 256, al = tb + 288;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        mma_ts_w(d, ah + k * 8, bd0 + 2 * k, idesc, 1);
        mma_ts_w(dc, al + k * 8, bd0 + 2 * k, idesc, 1);
        mma_ts_w(dc, ah + k * 8, bd0 + 512 + 2 * k, idesc, 1);
      }
    }
    if (threadIdx.x == 0) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (unsigned long long)(t1 - t0); stop = 1; }
  } else if (warp >= 2 && warp <= 5 && ld_on) {
    const uint32_t base = tb + ((uint32_t)((warp & 3) * 32) << 16) + 128;
    int i = 0;
    while (!stop) {
      uint32_t r[32];
      ld32(base + ((i++ * 32) & 63), r);
      acc += __uint_as_float(r[i & 31]);
    }
  } else if (warp >= 6 && warp <= 9 && st_on) {
    const uint32_t base = tb + ((uint32_t)((warp & 3) * 32) << 16) + 320;
    uint32_t r[32];
    for (int e = 0; e < 32; ++e) r[e] = e;
    int i = 0;
    while (!stop) {
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
          ::"r"(base + ((i++ * 32) & 127)), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
            "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
            "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
            "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  if (acc == 1234.5f) out[1] = 1;
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tb);
}

// shared-memory contention: warp 0 issues the 3xTF32 TS pattern while `nw` other warps stream
// 16-byte loads (mode 1) or stores (mode 2) through a separate 64 KB region
__global__ void k_smem_contend(int iters, int nw, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); stop = 0; }
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const int warp = threadIdx.x / 32;
  float acc = 0.f;
  float4* buf = reinterpret_cast<float4*>(sm + 65536);
  if (warp == 0) {
    const uint32_t idesc = make_idesc(FMT_TF32, 128, 64);
    const uint64_t bd0 = make_sdesc(smem_u32(sm) + 16384, 16, 1024, LAYOUT_SW128);
    const uint32_t d = tb, dc = tb + 64, ah = tb + 256, al = tb + 288;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        mma_ts_w(d, ah + k * 8, bd0 + 2 * k, idesc, 1);
        mma_ts_w(dc, al + k * 8, bd0 + 2 * k, idesc, 1);
        mma_ts_w(dc, ah + k * 8, bd0 + 512 + 2 * k, idesc, 1);
      }
    }
    if (threadIdx.x == 0) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (unsigned long long)(t1 - t0); stop = 1; }
  } else if (warp >= 1 && warp <= nw) {
    int i = threadIdx.x;
    while (!stop) {
      if (mode == 1) { const float4 v = buf[i & 4095]; acc += v.x; }
      else buf[i & 4095] = make_float4(acc, 1.f, 2.f, 3.f);
      i += 32 * nw;
    }
  }
  if (acc == 1234.5f) out[1] = 1;
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tb);
}

// commits between chunks: a tcgen05.commit to an mbarrier after every `per` chunks of 12 MMAs
__global__ void k_mma_commit(int iters, int per, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ uint64_t bar, cb[4];
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) mbar_init(&cb[i], 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const long long t0 = clock64();
  if (threadIdx.x < 32) {
    const uint32_t idesc = make_idesc(FMT_TF32, 128, 64);
    const uint64_t wd = make_sdesc(smem_u32(sm) + 16384, 16, 1024, LAYOUT_SW128);
    for (int i = 0; i < iters; ++i) {
      mma_3xtf32_ts_chunk_w(tb, tb + 64, tb + 256 + (i & 1) * 64, tb + 288 + (i & 1) * 64, wd, wd + 512, idesc, 1);
      if (per > 0 && (i % per) == per - 1) { mma_commit_w(&cb[i & 3]); mma_commit_w(&cb[(i + 1) & 3]); }
      if (per < 0) tc_fence_after();              // fence::after_thread_sync between chunks
      if (per < -1) tc_fence_before();
    }
    if (threadIdx.x == 0) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tb);
}

// ALU issue contention: warp 1 issues 3xTF32 TS chunks while `nw` other warps run dense
// independent integer/float work (no memory), like the transform and epilogue warps
__global__ void k_mma_alu(int iters, int nw, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); stop = 0; }
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0);
  if (nw < 0) {                 // non-zero operands: random-ish smem B and TMEM A
    for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
      reinterpret_cast<float*>(sm)[i] = __uint_as_float(0x3f800000u | ((i * 2654435761u) >> 9));
    fence_async_smem();
    if (warp < 4) {
      uint32_t v[32];
      for (int e = 0; e < 32; ++e) v[e] = 0x3f800000u | (((threadIdx.x * 37 + e) * 2654435761u) >> 9);
      const uint32_t ta = tb + ((uint32_t)((warp & 3) * 32) << 16);
      for (int c = 0; c < 512; c += 32)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                     "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                     ::"r"(ta + c), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                       "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
                       "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
                       "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
  }
  uint32_t x[8];
  for (int e = 0; e < 8; ++e) x[e] = threadIdx.x * 7 + e;
  if (warp == 1) {
    const uint32_t idesc = make_idesc(FMT_TF32, 128, 64);
    const uint64_t wd = make_sdesc(smem_u32(sm) + 16384, 16, 1024, LAYOUT_SW128);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
      mma_3xtf32_ts_chunk_w(tb, tb + 64, tb + 256 + (i & 1) * 64, tb + 288 + (i & 1) * 64, wd, wd + 512, idesc, 1);
    if (lane_id() == 0) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (lane_id() == 0) { out[0] = (unsigned long long)(t1 - t0); stop = 1; }
  } else if (warp >= 2 && warp < 2 + (nw < 0 ? 0 : nw)) {
    while (!stop) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] = ((x[e] + 0x1000u) & 0xFFFFE000u) ^ (x[(e + 1) & 7] >> 3);
    }
  }
  uint32_t acc = 0;
  for (int e = 0; e < 8; ++e) acc ^= x[e];
  if (acc == 0x12345u) out[1] = 1;
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tb);
}

// spin-wait contention: warp 1 issues 3xTF32 TS chunks with 2 commits per chunk (as the GEMM)
// while `nw` other warps spin in mbarrier.try_wait on a barrier that never completes
__global__ void k_mma_spin(int iters, int nw, int hint_ns, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ uint64_t bar, never, cb[4];
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&never, 1); for (int i = 0; i < 4; ++i) mbar_init(&cb[i], 1); fence_mbar_init(); stop = 0; }
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0);
  if (warp == 1) {
    const uint32_t idesc = make_idesc(FMT_TF32, 128, 64);
    const uint64_t wd = make_sdesc(smem_u32(sm) + 16384, 16, 1024, LAYOUT_SW128);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      mma_3xtf32_ts_chunk_w(tb, tb + 64, tb + 256 + (i & 1) * 64, tb + 288 + (i & 1) * 64, wd, wd + 512, idesc, 1);
      mma_commit_w(&cb[i & 3]);
      mma_commit_w(&cb[(i + 1) & 3]);
    }
    if (lane_id() == 0) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (lane_id() == 0) { out[0] = (unsigned long long)(t1 - t0); stop = 1; }
  } else if (warp >= 2 && warp < 2 + nw) {
    while (!stop) {
      uint32_t ok;
      if (hint_ns > 0)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0, %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&never)), "r"(hint_ns) : "memory");
      else
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&never)) : "memory");
      if (ok) break;
    }
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tb);
}

// MMA issue with operands that are runtime values (kernel parameters offset by a loop counter
// and a value loaded from shared memory), as in the real kernels
__global__ void k_mma_rt(int iters, uint32_t doff, uint32_t aoff, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const long long t0 = clock64();
  if (threadIdx.x < 32) {
    const uint32_t idesc = make_idesc(FMT_TF32, 128, 64);
    const uint32_t base = tb;
    for (int i = 0; i < iters; ++i) {
      const uint32_t j = (uint32_t)i & 1;
      const uint64_t wd = make_sdesc(smem_u32(sm) + 16384 + j * 8192, 16, 1024, LAYOUT_SW128);
      const uint32_t d = base + doff + j * 64, dc = d + 128, ah = base + aoff + j * 64, al = ah + 32;
      mma_3xtf32_ts_chunk_w(d, dc, ah, al, wd, wd + 512, idesc, 1);
    }
    if (threadIdx.x == 0) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tb);
}

__global__ void k_tmem_ld64(int nwarps, int iters, unsigned long long* out, float* sink) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tb);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  float acc = 0.f;
  const long long t0 = clock64();
  if (warp < nwarps) {
    const uint32_t base = tb + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp / 4) * 256);
    for (int i = 0; i < iters; i += 2) {
      uint32_t r[64], q[64];
      ld128nw(base + ((i * 64) & 255), r);
      ld128nw(base + ((i * 64 + 64) & 255), q);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc += __uint_as_float(r[i & 63]) + __uint_as_float(q[(i + 1) & 63]);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  if (acc == 1234.5f) sink[0] = acc;
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

__global__ void k_tmem_ld(int nwarps, int iters, unsigned long long* out, float* sink) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tb);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  float acc = 0.f;
  const long long t0 = clock64();
  if (warp < nwarps) {
    const uint32_t base = tb + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp / 4) * 256);
    for (int i = 0; i < iters; ++i) {
      uint32_t r[32];
      ld32(base + ((i * 32) & 255), r);
      acc += __uint_as_float(r[i & 31]);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  if (acc == 1234.5f) sink[0] = acc;
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

// mode 0: SS (A, B in smem, SW128 K-major); mode 1: TS (A in TMEM cols [256, 320))
// nacc independent accumulators (columns 0, 64, ...) written round-robin
__global__ void k_mma(int mode, int N, int iters, unsigned long long* out, int nacc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc(FMT_TF32, 128, N);
    const uint32_t a0 = smem_u32(sm), b0 = a0 + 16384;
    const uint64_t ad0 = make_sdesc(a0, 16, 1024, LAYOUT_SW128), bd0 = make_sdesc(b0, 16, 1024, LAYOUT_SW128);
    const uint32_t stride = (uint32_t)(N > 64 ? N : 64);
    const long long t0 = clock64();
    if (nacc == 1) {
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (mode == 0) mma_tf32(tb, ad0 + 2 * k, bd0 + 2 * k, idesc, 1);
          else mma_ts(tb, tb + 448 + k * 8, bd0 + 2 * k, idesc, 1);
        }
      }
    } else if (nacc == 2) {
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t dd = tb + (k & 1) * stride;
          if (mode == 0) mma_tf32(dd, ad0 + 2 * k, bd0 + 2 * k, idesc, 1);
          else mma_ts(dd, tb + 448 + k * 8, bd0 + 2 * k, idesc, 1);
        }
      }
    } else {
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t dd = tb + k * stride;
          if (mode == 0) mma_tf32(dd, ad0 + 2 * k, bd0 + 2 * k, idesc, 1);
          else mma_ts(dd, tb + 448 + k * 8, bd0 + 2 * k, idesc, 1);
        }
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    out[0] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tb);
}

__global__ void k_smem(int nwarps, int iters, unsigned long long* out, float* sink) {
  extern __shared__ __align__(16) float4 s4[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s4[i] = make_float4(i, 0, 0, 0);
  __syncthreads();
  float acc = 0.f;
  const long long t0 = clock64();
  if ((int)(threadIdx.x / 32) < nwarps)
    for (int i = 0; i < iters; ++i) {
      const float4 v = s4[(threadIdx.x + i * 32) & 8191];
      acc += v.x;
    }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  if (acc == 1234.5f) sink[0] = acc;
}

int main() {
  unsigned long long* d; float* sink; unsigned long long h;
  cudaMalloc(&d, 8); cudaMalloc(&sink, 4);
  for (int nw : {1, 2, 4, 8}) {
    const int it = 4096;
    k_tmem_ld<<<1, 256>>>(nw, it, d, sink);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("tmem ld x32: %d warps: %.1f B/cycle (%.0f cyc per 4KB warp-load)\n", nw,
           (double)nw * it * 4096 / h, (double)h / it);
  }
  cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int mode : {0, 1})
    for (int N : {64, 128})
      for (int nacc : {1, 2, 4}) {
        if ((N > 64 ? N : 64) * nacc > 448) continue;
        const int it = 2048;
        k_mma<<<1, 128, 64 * 1024>>>(mode, N, it, d, nacc);
        cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("mma tf32 %s M=128 N=%d K=8 nacc=%d: %.1f cyc/mma (floor %d) %s\n", mode ? "TS" : "SS", N, nacc,
               (double)h / (4.0 * it), 128 * N / 256, cudaGetErrorString(e));
      }
  cudaFuncSetAttribute(k_mma_w, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int mode : {0, 1})
    for (int N : {64, 128, 256})
      for (int nacc : {1, 2, 4}) {
        if ((N > 64 ? N : 64) * nacc > 448) continue;
        const int it = 2048;
        k_mma_w<<<1, 128, 64 * 1024>>>(mode, N, it, d, nacc);
        cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("warp-issued mma tf32 %s M=128 N=%d nacc=%d: %.1f cyc/mma (floor %d) %s\n", mode ? "TS" : "SS", N, nacc,
               (double)h / (4.0 * it), 128 * N / 256, cudaGetErrorString(e));
      }
  cudaFuncSetAttribute(k_mma_mw<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(k_mma_mw<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int ts = 0; ts < 2; ++ts)
    for (int N : {64, 128})
      for (int nw : {1, 2}) {
        const int it = 2048;
        if (ts) k_mma_mw<true><<<1, 128, 64 * 1024>>>(N, it, d, nw);
        else k_mma_mw<false><<<1, 128, 64 * 1024>>>(N, it, d, nw);
        cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("mma tf32 %s N=%d issuers=%d: %.1f cyc per mma (all issuers) %s\n", ts ? "TS" : "SS", N, nw,
               (double)h / (4.0 * it * nw), cudaGetErrorString(e));
      }
  cudaFuncSetAttribute(k_mma_3x<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(k_mma_3x<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int mode = 0; mode < 2; ++mode) {
    const int it = 2048;
    if (mode == 0) k_mma_3x<0><<<1, 128, 64 * 1024>>>(it, d);
    else k_mma_3x<1><<<1, 128, 64 * 1024>>>(it, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("3xTF32 TS pattern, %s: %.1f cyc per mma\n", mode == 0 ? "main + corr accumulators" : "one accumulator",
           (double)h / (12.0 * it));
  }
  cudaFuncSetAttribute(k_contend, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int cfg = 0; cfg < 4; ++cfg) {
    const int it = 4096;
    k_contend<<<1, 320, 64 * 1024>>>(it, cfg & 1, cfg >> 1, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("3xTF32 TS MMA with TMEM ld %s, st %s: %.1f cyc per mma\n", (cfg & 1) ? "on " : "off", (cfg >> 1) ? "on " : "off",
           (double)h / (12.0 * it));
  }
  cudaFuncSetAttribute(k_smem_contend, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  for (int mode = 1; mode <= 2; ++mode)
    for (int nw : {2, 4, 8}) {
      const int it = 4096;
      k_smem_contend<<<1, 320, 128 * 1024>>>(it, nw, mode, d);
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("3xTF32 TS MMA with %d warps of smem %s: %.1f cyc per mma\n", nw, mode == 1 ? "loads" : "stores",
             (double)h / (12.0 * it));
    }
  cudaFuncSetAttribute(k_mma_commit, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int per : {0, 1, 2, 4, -1, -2}) {
    const int it = 4096;
    k_mma_commit<<<1, 128, 64 * 1024>>>(it, per, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("3xTF32 TS chunks with 2 commits every %d chunks: %.1f cyc per mma\n", per, (double)h / (12.0 * it));
  }
  cudaFuncSetAttribute(k_mma_alu, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int nw : {0, 8, -1}) {
    const int it = 4096;
    k_mma_alu<<<1, 320, 64 * 1024>>>(it, nw, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("3xTF32 TS chunks with %d dense-ALU warps (-1: nonzero operands): %.1f cyc per mma\n", nw, (double)h / (12.0 * it));
  }
  cudaFuncSetAttribute(k_mma_spin, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int cfg = 0; cfg < 5; ++cfg) {
    const int nw = cfg == 0 ? 0 : (cfg < 3 ? 4 : 8), hint = (cfg == 2 || cfg == 4) ? 20000 : 0;
    const int it = 4096;
    k_mma_spin<<<1, 320, 64 * 1024>>>(it, nw, hint, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("3xTF32 TS chunks + commits, %d warps spinning in try_wait (hint %d ns): %.1f cyc per mma\n", nw, hint,
           (double)h / (12.0 * it));
  }
  cudaFuncSetAttribute(k_mma_rt, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  {
    const int it = 4096;
    k_mma_rt<<<1, 128, 64 * 1024>>>(it, 0, 384, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("3xTF32 TS chunk, runtime operands: %.1f cyc per mma\n", (double)h / (12.0 * it));
  }
  for (int nw : {1, 4, 8}) {
    const int it = 4096;
    k_tmem_ld64<<<1, 256>>>(nw, it, d, sink);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("tmem ld x64 pairs: %d warps: %.1f B/cycle\n", nw, (double)nw * it * 8192 / h);
  }
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  for (int nw : {4, 8, 16}) {
    const int it = 8192;
    k_smem<<<1, 512, 128 * 1024>>>(nw, it, d, sink);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("smem ld.v4: %d warps: %.1f B/cycle\n", nw, (double)nw * it * 512 / h);
  }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
