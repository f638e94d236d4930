// Fused persistent bank kernel (SISO channels, m = 64, fp32 mode / 3xTF32): the whole cascade
// of PAPER.md:185-229 for every channel in ONE launch, with the state kept on chip.
//
// Per sequence (channel c, batch b) with effective order Ne >= 7 the path is the one of
// bank_tc.cu, level by level (v^(j) = state after stages 0..j-1):
//   head   v^(7)_l   = sum_{i<128} (Abar^i Bbar) u_{l-i}           (stages 0..6 + Bbar u, R22)
//   stage  v^(j+1)_l = v^(j)_l + P_j v^(j)_{l-2^j},  j = 7..Ne-1
//   tail   y_l       = c.v^(Ne)_l + (c P_Ne).v^(Ne)_{l-2^Ne} + d u_l (stage Ne fused with y)
// For j >= 7 the shift 2^j is a whole number of 128-step tiles, so the shifted operand of tile t
// at level j is exactly tile t - 2^(j-7).
//
// Schedule. A sequence is cut into chunks of T <= 6 tiles; chunks are dealt round-robin to
// persistent CTAs (one per SM). A CTA keeps the states of its chunk's tiles in TMEM (64 columns
// per tile) across all levels: the residual v^(j)_l never leaves the SM. The only traffic per
// tile and level is the tile's publication (32 KB, TMA store) for the one consumer tile
// t + 2^(j-7) and that consumer's TMA load of it, both through L2; the consumer then discards
// the lines (discard.global.L2), so the dead data is never written back to HBM. Publication is
// tracked by per-tile flags: flag[slot][t] = (q << 5) | j once level j of tile t of sequence q
// is visible. Publication buffers have one plane per level (no write-after-read hazards inside a
// sequence) and S sequence slots reused round-robin; a chunk of sequence q >= S starts only after
// every chunk of sequence q - S completed (done[] counters). Every wait is on a lower chunk index
// or an earlier op of the same chunk, and chunks are processed in increasing index per CTA, so the
// smallest unfinished chunk can always progress (no deadlock with all CTAs resident).
//
// Roles (352 threads):
//   warp 0     producer: Krylov weights (bulk copy), P_j hi/lo (TMA), flag waits, TMA loads of
//              shifted tiles into a ring of 16 KB K-chunk units
//   warp 1     MMA issuer (tcgen05 kind::tf32, M=128, N=64): head K=128 (Toeplitz operand in
//              shared memory, as bank_head_ws.cu), stage K=64; hi.hi + lo.hi + hi.lo into one
//              TMEM accumulator (double-buffered); the epilogue adds it to the state (RN)
//   warps 2-5  epilogue (lane = time row): state += accumulator (round to nearest), published
//              halves into two SW128 staging slots; tail dot products and y
//   warp 10    store: TMA stores of the staged halves; releases a tile's flag once its stores are
//              complete (up to PD tiles in flight), so store latency stays off the epilogue
//   warps 6-9  transform: Toeplitz operand Z from u (head), hi/lo split of landed units (stage)
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "sm100.cuh"
#include "bank_tc.cuh"
#include "mimo_tc.cuh"

namespace casc {
using namespace sm100;

namespace {
constexpr int TM = 128;                     // time rows per tile
constexpr int NA = 6;                       // fp32 units (16 KB K-chunks of a shifted tile)
constexpr int NAU = 2;                      // TMEM A units (tf32 hi | lo of one K-chunk)
constexpr uint32_t UNIT = 16384;
constexpr uint32_t OFF_A = 0;
constexpr uint32_t OFF_W = OFF_A + NA * UNIT;        // 64 KB: Krylov hi | lo, or P_j in halves
constexpr uint32_t OFF_Z = OFF_W + 65536;            // 2 slots x (hi 4 KB | lo 4 KB)
constexpr uint32_t OFF_STG = OFF_Z + 16384;          // 2 x 16 KB publication staging slots
constexpr uint32_t SMEM_USED = OFF_STG + 2 * UNIT;
// the dynamic region is declared 1024-aligned (the static part is padded to keep it so; checked
// at run time), so no alignment slack is requested
constexpr size_t SMEM_BYTES = SMEM_USED;
constexpr int STORE_WARP = 10;
constexpr int THREADS = 32 * (STORE_WARP + 1);
constexpr int PD = 4;                                // published tiles in flight per CTA
constexpr int TMAX = 4;                              // tiles per chunk (TMEM state slots)
constexpr uint32_t ACC0 = TMAX * 64;                 // TMEM: states [0, 256), two accumulators,
constexpr uint32_t AU0 = ACC0 + 2 * 64;              // then NAU A units of 64 columns (hi | lo)

__device__ __forceinline__ void named_sync_f(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];"
               ::"l"(map), "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void commit_f() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_read_f() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
template <int N>
__device__ __forceinline__ void wait_all_f() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ uint32_t ld_acquire(const unsigned* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void discard_line(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void tmem_ld32f(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32f(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
        "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
        "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ldf() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_stf() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

struct FusedMaps {
  CUtensorMap pub;        // [S*NL planes][ntiles*128][64] fp32, box {32, 128, 1}, SW128
  CUtensorMap P;          // pack fp32 planes [n*(N_max+1)*2][64][64], box {32, 64, 1}, SW128
};

struct Chunk {
  int q, c, seq, Ne, t0, nt, slot;
};
__device__ __forceinline__ Chunk chunk_of(int64_t g, const BankFusedArg& a) {
  Chunk k;
  k.q = (int)(g / a.nchunk);
  const int ci = (int)(g % a.nchunk);
  const int li = k.q / a.batch, b = k.q % a.batch;
  k.c = a.order[li];
  k.seq = k.c * a.batch + b;
  k.Ne = a.Neff[k.c];
  k.t0 = ci * a.T;
  k.nt = min(a.T, a.ntiles - k.t0);
  k.slot = k.q % a.S;
  return k;
}
__device__ __forceinline__ int64_t tshift(int j) { return (int64_t)1 << (j - 7); }   // tiles
// number of tiles of a chunk that publish a level (head: level 7; stage j: level j+1)
__device__ __forceinline__ int publishes_in_chunk(const Chunk& k, const BankFusedArg& a) {
  int n = 0;
  for (int j = 7; j <= k.Ne; ++j)
    for (int i = 0; i < k.nt; ++i) n += ((int64_t)(k.t0 + i) + tshift(j) < a.ntiles) ? 1 : 0;
  return n;
}
struct StgDesc {
  int plane, row0, col;
  unsigned* flag;                // set on the second half of a tile: release after both stores
  uint32_t val;
};
}  // namespace

__global__ void __launch_bounds__(THREADS, 1) bank_fused_kernel(const __grid_constant__ FusedMaps maps, BankFusedArg a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023u) __trap();          // SW128 tiles need 1024-B alignment
  uint8_t* smem = smem_raw;
  uint8_t* sA = smem + OFF_A;
  uint8_t* sW = smem + OFF_W;
  float* sZ = reinterpret_cast<float*>(smem + OFF_Z);
  uint8_t* sSTG = smem + OFF_STG;
  __shared__ float sCW[128];                         // c | w of the chunk's channel (tail)
  __shared__ StgDesc stg_desc[2];
  __shared__ uint64_t afull[NA], aempty[NA], auready[NAU], aufree[NAU], wfull[2], wfree[2], zfull[2], zempty[2],
      accfull[2], accempty[2], stg_full[2], stg_empty[2], tready[NA];
  __shared__ uint32_t tmem_base;

  // warp index broadcast from lane 0: provably warp-uniform, so role branches are uniform control
  // flow and ptxas keeps role-local uniform values (descriptors, TMEM addresses) in uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  // optional wait-time accounting (a.dbg != null): 4 counters per role, clock64 cycles
  unsigned long long dacc[4] = {0, 0, 0, 0};
  const long long t_start = clock64();
#define TW(slot, stmt)                                   \
  do {                                                   \
    if (a.dbg) {                                         \
      const long long t0_ = clock64();                   \
      stmt;                                              \
      dacc[slot] += (unsigned long long)(clock64() - t0_); \
    } else {                                             \
      stmt;                                              \
    }                                                    \
  } while (0)
  if (threadIdx.x == 0) {
    for (int s = 0; s < NA; ++s) { mbar_init(&afull[s], 1); mbar_init(&aempty[s], 1); mbar_init(&tready[s], 1); }
    for (int s = 0; s < NAU; ++s) { mbar_init(&auready[s], 128); mbar_init(&aufree[s], 1); }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&wfull[s], 1); mbar_init(&wfree[s], 1);
      mbar_init(&zfull[s], 128); mbar_init(&zempty[s], 1);
      mbar_init(&accfull[s], 1); mbar_init(&accempty[s], 128);
      mbar_init(&stg_full[s], 128); mbar_init(&stg_empty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&tmem_base);
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.pub) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.P) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  const int64_t pub_plane_floats = (int64_t)a.ntiles * TM * 64;

  if (warp == 0) {
    // ================================================================== producer
    if (lane == 0) {
      uint32_t na = 0, wu[2] = {0, 0};
      for (int64_t g = blockIdx.x; g < a.total_chunks; g += gridDim.x) {
        const Chunk k = chunk_of(g, a);
        TW(0, mbar_wait(&wfree[0], (wu[0] & 1) ^ 1));
        TW(0, mbar_wait(&wfree[1], (wu[1] & 1) ^ 1));
        const float* img = a.krimg + (int64_t)k.c * 16384;
        mbar_arrive_expect_tx(&wfull[0], 32768);
        bulk_g2s(sW, img, 32768, &wfull[0]);
        mbar_arrive_expect_tx(&wfull[1], 32768);
        bulk_g2s(sW + 32768, img + 8192, 32768, &wfull[1]);
        ++wu[0];
        ++wu[1];
        for (int j = 7; j <= k.Ne; ++j) {
          if (j < k.Ne) {                                   // P_j hi | lo into half (j-7)&1
            const int h = (j - 7) & 1;
            TW(0, mbar_wait(&wfree[h], (wu[h] & 1) ^ 1));
            mbar_arrive_expect_tx(&wfull[h], 32768);
            const int plane = k.c * a.planes_per_ch + 2 * j;
            uint8_t* dst = sW + h * 32768;
            tma_load3(dst, &maps.P, &wfull[h], 0, 0, plane);
            tma_load3(dst + 8192, &maps.P, &wfull[h], 32, 0, plane);
            tma_load3(dst + 16384, &maps.P, &wfull[h], 0, 0, plane + 1);
            tma_load3(dst + 24576, &maps.P, &wfull[h], 32, 0, plane + 1);
            ++wu[h];
          }
          const uint32_t need = ((uint32_t)k.q << 5) | (uint32_t)j;
          for (int i = 0; i < k.nt; ++i) {
            const int64_t ts = (int64_t)(k.t0 + i) - tshift(j);
            if (ts < 0) continue;
            const unsigned* f = a.flags + (int64_t)k.slot * a.ntiles + ts;
            if (ld_acquire(f) < need) {
              TW(1, while (ld_acquire(f) < need) __nanosleep(64));
            }
            fence_async_global();
            for (int kc = 0; kc < 2; ++kc, ++na) {
              const int s = (int)(na % NA);
              TW(2, mbar_wait(&aempty[s], ((na / NA) & 1) ^ 1));
              mbar_arrive_expect_tx(&afull[s], UNIT);
              tma_load3(sA + s * UNIT, &maps.pub, &afull[s], kc * 32, (int)(ts * TM), k.slot * a.NL + (j - 7));
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================================================================== MMA issuer (whole warp)
    {
      const uint32_t idesc = make_idesc(FMT_TF32, TM, 64);
      uint32_t nz = 0, na = 0, nau = 0, nacc = 0, wu[2] = {0, 0};
      const uint32_t bh = smem_u32(sW), bl = bh + 32768;
      for (int64_t g = blockIdx.x; g < a.total_chunks; g += gridDim.x) {
        const Chunk k = chunk_of(g, a);
        TW(0, mbar_wait(&wfull[0], wu[0] & 1));
        TW(0, mbar_wait(&wfull[1], wu[1] & 1));
        tc_fence_after();
        for (int i = 0; i < k.nt; ++i, ++nz, ++nacc) {      // head: K = 128 Toeplitz GEMM
          const int zs = (int)(nz & 1), ac = (int)(nacc & 1);
          TW(1, mbar_wait(&zfull[zs], (nz >> 1) & 1));
          TW(2, mbar_wait(&accempty[ac], ((nacc >> 1) & 1) ^ 1));
          tc_fence_after();
          const uint32_t d = tbase + ACC0 + ac * 64;
          const uint32_t zh = smem_u32(sZ + zs * 2048), zl = zh + 4096;
          const uint64_t azh0 = make_sdesc(zh, 64, 128, LAYOUT_NONE), azl0 = make_sdesc(zl, 64, 128, LAYOUT_NONE);
          const uint64_t bdh0 = make_sdesc(bh, 64 * 16, 128, LAYOUT_NONE), bdl0 = make_sdesc(bl, 64 * 16, 128, LAYOUT_NONE);
#pragma unroll
          for (int ks = 0; ks < 16; ++ks) {          // descriptor start field advances by bytes >> 4
            mma_tf32_w(d, azh0 + ks * 8, bdh0 + ks * 128, idesc, ks > 0);
            mma_tf32_w(d, azl0 + ks * 8, bdh0 + ks * 128, idesc, 1);
            mma_tf32_w(d, azh0 + ks * 8, bdl0 + ks * 128, idesc, 1);
          }
          mma_commit_w(&zempty[zs]);
          mma_commit_w(&accfull[ac]);
        }
        mma_commit_w(&wfree[0]);
        mma_commit_w(&wfree[1]);
        ++wu[0];
        ++wu[1];
        for (int j = 7; j <= k.Ne; ++j) {
          const int h = (j - 7) & 1;
          if (j < k.Ne) {
            TW(0, mbar_wait(&wfull[h], wu[h] & 1));
            tc_fence_after();
          }
          for (int i = 0; i < k.nt; ++i) {
            const int64_t ts = (int64_t)(k.t0 + i) - tshift(j);
            if (ts < 0) continue;
            if (j == k.Ne) {                               // tail units: consumed by the epilogue
              na += 2;
              continue;
            }
            const int ac = (int)(nacc & 1);
            TW(2, mbar_wait(&accempty[ac], ((nacc >> 1) & 1) ^ 1));
            tc_fence_after();
            const uint32_t d = tbase + ACC0 + ac * 64;
            bool first = true;
            for (int kc = 0; kc < 2; ++kc, ++na, ++nau) {
              const int au = (int)(nau % NAU);
              TW(3, mbar_wait(&auready[au], (nau / NAU) & 1));
              tc_fence_after();
              const uint32_t ah = tbase + AU0 + au * 64, al = ah + 32;
              const uint64_t wd0 = make_sdesc(smem_u32(sW + h * 32768 + kc * 8192), 16, 1024, LAYOUT_SW128);
              const uint64_t wl0 = wd0 + (16384 >> 4);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {           // A (shifted state) from TMEM: no smem reads
                mma_tf32_ts_w(d, ah + kk * 8, wd0 + 2 * kk, idesc, first ? 0u : 1u);
                mma_tf32_ts_w(d, al + kk * 8, wd0 + 2 * kk, idesc, 1u);
                mma_tf32_ts_w(d, ah + kk * 8, wl0 + 2 * kk, idesc, 1u);
                first = false;
              }
              mma_commit_w(&aufree[au]);
            }
            mma_commit_w(&accfull[ac]);
            ++nacc;
          }
          if (j < k.Ne) {
            mma_commit_w(&wfree[h]);
            ++wu[h];
          }
        }
      }
    }
  } else if (warp >= 6 && warp < STORE_WARP) {
    // ================================================================== transform
    const int tt = threadIdx.x - 192;
    const int trow = (warp & 3) * 32 + lane;        // TMEM lane this warp may access
    const uint32_t trow_t = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t nz = 0, na = 0, nau = 0, ntr = 0;
    for (int64_t g = blockIdx.x; g < a.total_chunks; g += gridDim.x) {
      const Chunk k = chunk_of(g, a);
      if (k.q >= a.S) {                 // slot reuse: sequence q - S must be complete
        if (tt == 0) {
          const unsigned* dn = a.done + (k.q - a.S);
          TW(0, while (ld_acquire(dn) < (uint32_t)a.nchunk) __nanosleep(128));
        }
        named_sync_f(2, 128);
      }
      const float* u = a.u + (int64_t)k.seq * a.L;
      // Z-row w = (u[t0 - 127 + w + e], e = 0..3); rows >= 252 are never read (zeroed)
      float zr[2][4];
      auto load_u = [&](int i) {
        const int64_t base = (int64_t)(k.t0 + i) * TM - 127;
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int w = tt + 128 * rr;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int64_t x = base + w + e;
            zr[rr][e] = (w < 252 && x >= 0 && x < a.L) ? __ldg(u + x) : 0.f;
          }
        }
      };
      load_u(0);
      for (int i = 0; i < k.nt; ++i, ++nz) {
        const int zs = (int)(nz & 1);
        TW(1, mbar_wait(&zempty[zs], ((nz >> 1) & 1) ^ 1));
        float* zh = sZ + zs * 2048;
        float* zl = zh + 1024;
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int w = tt + 128 * rr;
          const float4 z = make_float4(zr[rr][0], zr[rr][1], zr[rr][2], zr[rr][3]);
          const float4 h = tf32_hi4(z);
          *reinterpret_cast<float4*>(zh + w * 4) = h;
          *reinterpret_cast<float4*>(zl + w * 4) = tf32_lo4(z, h);
        }
        fence_async_smem();
        mbar_arrive(&zfull[zs]);
        if (i + 1 < k.nt) load_u(i + 1);
      }
      for (int j = 7; j <= k.Ne; ++j) {
        const int64_t plane = (int64_t)k.slot * a.NL + (j - 7);
        for (int i = 0; i < k.nt; ++i) {
          const int64_t ts = (int64_t)(k.t0 + i) - tshift(j);
          if (ts < 0) continue;
          if (j == k.Ne) {                 // tail units: confirm landing for the epilogue
            for (int kc = 0; kc < 2; ++kc, ++na, ++ntr) {
              TW(2, mbar_wait(&afull[(int)(na % NA)], (na / NA) & 1));
              if (tt == 0) mbar_arrive(&tready[ntr % NA]);
            }
            continue;
          }
          for (int kc = 0; kc < 2; ++kc, ++na, ++nau) {
            const int s = (int)(na % NA), au = (int)(nau % NAU);
            TW(2, mbar_wait(&afull[s], (na / NA) & 1));
            // this thread's row of the landed K-chunk (SW128: 16-B chunk c at (c ^ (row % 8)) * 16)
            const uint8_t* rr = sA + s * UNIT + trow * 128;
            uint32_t hv[32], lv[32];
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
              const float4 v = *reinterpret_cast<const float4*>(rr + ((cc ^ (trow & 7)) * 16));
              const float4 hh = tf32_hi4(v), ll = tf32_lo4(v, hh);
              hv[4 * cc] = __float_as_uint(hh.x); hv[4 * cc + 1] = __float_as_uint(hh.y);
              hv[4 * cc + 2] = __float_as_uint(hh.z); hv[4 * cc + 3] = __float_as_uint(hh.w);
              lv[4 * cc] = __float_as_uint(ll.x); lv[4 * cc + 1] = __float_as_uint(ll.y);
              lv[4 * cc + 2] = __float_as_uint(ll.z); lv[4 * cc + 3] = __float_as_uint(ll.w);
            }
            if (a.discard)                              // line = half row (this K-chunk) of row trow
              discard_line(a.pub + plane * pub_plane_floats + (ts * TM + trow) * 64 + kc * 32);
            named_sync_f(2, 128);                       // every row read: the smem unit is free
            if (tt == 0) mbar_arrive(&aempty[s]);
            TW(3, mbar_wait(&aufree[au], ((nau / NAU) & 1) ^ 1));
            tc_fence_after();
            tmem_st32f(trow_t + AU0 + au * 64, hv);
            tmem_st32f(trow_t + AU0 + au * 64 + 32, lv);
            tmem_wait_stf();
            tc_fence_before();
            mbar_arrive(&auready[au]);
          }
        }
      }
    }
  } else if (warp == STORE_WARP) {
    // ================================================================== store warp
    // Issues the TMA stores of published half tiles and releases each tile's flag once both of
    // its stores are complete, keeping up to PD tiles in flight; whenever no staging slot is
    // ready it drains completions instead (it never blocks while holding a release it could make).
    if (lane == 0) {
      unsigned* pf[PD + 1];
      uint32_t pv[PD + 1];
      int np = 0;
      auto release_oldest = [&]() {         // oldest pending tile: its 2 groups are the oldest
        switch (np) {                        // groups; 2*(np-1) younger groups may stay pending
          case 1: wait_all_f<0>(); break;
          case 2: wait_all_f<2>(); break;
          case 3: wait_all_f<4>(); break;
          case 4: wait_all_f<6>(); break;
          default: wait_all_f<8>(); break;
        }
        fence_async_global();
        st_release(pf[0], pv[0]);
        for (int i = 1; i < np; ++i) { pf[i - 1] = pf[i]; pv[i - 1] = pv[i]; }
        --np;
      };
      uint32_t nh = 0;
      int unread = -1;                        // staging slot whose store may still be reading it
      for (int64_t g = blockIdx.x; g < a.total_chunks; g += gridDim.x) {
        const Chunk k = chunk_of(g, a);
        const int n_pub = publishes_in_chunk(k, a);
        for (int p = 0; p < 2 * n_pub; ++p, ++nh) {
          const int s = (int)(nh & 1);
          const uint32_t par = (nh >> 1) & 1;
          while (!mbar_try(&stg_full[s], par)) {
            if (unread >= 0) {                        // idle: free the last slot first
              TW(1, wait_read_f<0>());
              mbar_arrive(&stg_empty[unread]);
              unread = -1;
            } else if (np > 0) {
              TW(2, release_oldest());
            } else {
              TW(0, mbar_wait(&stg_full[s], par));
              break;
            }
          }
          const StgDesc d = stg_desc[s];
          tma_store3(&maps.pub, sSTG + s * UNIT, d.col, d.row0, d.plane);
          commit_f();
          if (unread >= 0) {                          // the other slot's store has read its data
            TW(1, wait_read_f<1>());
            mbar_arrive(&stg_empty[unread]);
          }
          unread = s;
          if (d.flag) {
            pf[np] = d.flag;
            pv[np] = d.val;
            ++np;
            if (np > PD) release_oldest();
          }
        }
      }
      while (np > 0) release_oldest();
      wait_all_f<0>();
    }
  } else {
    // ================================================================== epilogue (warps 2-5)
    const int q4 = warp & 3, row = q4 * 32 + lane;
    const bool leader = (warp == 2 && lane == 0);
    const uint32_t lrow = tbase + ((uint32_t)(q4 * 32) << 16);
    uint32_t na = 0, nacc = 0, nh = 0, ntr = 0;
    // one 32-column half of this row -> staging slot (SW128) -> store warp
    auto publish_half = [&](const uint32_t* v, int hh, int64_t plane, int t, unsigned* flag, uint32_t val) {
      const int s = (int)(nh & 1);
      TW(1, mbar_wait(&stg_empty[s], ((nh >> 1) & 1) ^ 1));
      uint8_t* rr = sSTG + s * UNIT + row * 128;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc)
        *reinterpret_cast<uint4*>(rr + ((cc ^ (row & 7)) * 16)) =
            make_uint4(v[4 * cc], v[4 * cc + 1], v[4 * cc + 2], v[4 * cc + 3]);
      if (leader) {
        StgDesc d;
        d.plane = (int)plane;
        d.row0 = t * TM;
        d.col = hh * 32;
        d.flag = hh == 1 ? flag : nullptr;
        d.val = val;
        stg_desc[s] = d;
      }
      fence_async_smem();
      mbar_arrive(&stg_full[s]);
      ++nh;
    };
    for (int64_t g = blockIdx.x; g < a.total_chunks; g += gridDim.x) {
      const Chunk k = chunk_of(g, a);
      unsigned* fl = a.flags + (int64_t)k.slot * a.ntiles;
      const uint32_t qtag = (uint32_t)k.q << 5;
      // ---- head: state = accumulator; publish level 7 for tile t + 1
      for (int i = 0; i < k.nt; ++i, ++nacc) {
        const int t = k.t0 + i, ac = (int)(nacc & 1);
        TW(0, mbar_wait(&accfull[ac], (nacc >> 1) & 1));
        tc_fence_after();
        const bool pub = t + 1 < a.ntiles;
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t m[32];
          tmem_ld32f(lrow + ACC0 + ac * 64 + hh * 32, m);
          tmem_wait_ldf();
          tmem_st32f(lrow + i * 64 + hh * 32, m);
          if (hh == 1) {
            tc_fence_before();
            mbar_arrive(&accempty[ac]);
          }
          if (pub) publish_half(m, hh, (int64_t)k.slot * a.NL, t, fl + t, qtag | 7u);
        }
        tmem_wait_stf();
      }
      // ---- stages j = 7 .. Ne-1: state += P_j v_{t - 2^(j-7)}; publish level j+1
      for (int j = 7; j < k.Ne; ++j) {
        const int64_t plane = (int64_t)k.slot * a.NL + (j + 1 - 7);
        for (int i = 0; i < k.nt; ++i) {
          const int t = k.t0 + i;
          const bool has = (int64_t)t - tshift(j) >= 0;
          const bool pub = (int64_t)t + tshift(j + 1) < a.ntiles;
          const int ac = (int)(nacc & 1);
          if (has) {
            na += 2;
            TW(0, mbar_wait(&accfull[ac], (nacc >> 1) & 1));
            tc_fence_after();
          }
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t s[32];
            tmem_ld32f(lrow + i * 64 + hh * 32, s);
            if (has) {
              uint32_t m[32];
              tmem_ld32f(lrow + ACC0 + ac * 64 + hh * 32, m);
              tmem_wait_ldf();
#pragma unroll
              for (int e = 0; e < 32; ++e) s[e] = __float_as_uint(__uint_as_float(s[e]) + __uint_as_float(m[e]));
              tmem_st32f(lrow + i * 64 + hh * 32, s);
              if (hh == 1) {
                tc_fence_before();
                mbar_arrive(&accempty[ac]);
              }
            } else {
              tmem_wait_ldf();
            }
            if (pub) publish_half(s, hh, plane, t, fl + t, qtag | (uint32_t)(j + 1));
          }
          if (has) {
            tmem_wait_stf();
            ++nacc;
          }
        }
      }
      // ---- tail: y = c.v + w.v_{t - 2^(Ne-7)} + d u
      named_sync_f(1, 128);
      sCW[row] = row < 64 ? a.cvec[(int64_t)k.c * 64 + row] : a.wvec[(int64_t)k.c * 64 + row - 64];
      const float dval = a.dvec[k.c];
      named_sync_f(1, 128);
      const int64_t tplane = (int64_t)k.slot * a.NL + (k.Ne - 7);
      for (int i = 0; i < k.nt; ++i) {
        const int t = k.t0 + i;
        const int64_t ts = (int64_t)t - tshift(k.Ne);
        float yv = 0.f;
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t s[32];
          tmem_ld32f(lrow + i * 64 + hh * 32, s);
          tmem_wait_ldf();
#pragma unroll
          for (int e = 0; e < 32; ++e) yv = fmaf(sCW[hh * 32 + e], __uint_as_float(s[e]), yv);
        }
        if (ts >= 0) {
          for (int kc = 0; kc < 2; ++kc, ++na) {
            const int s = (int)(na % NA);
            TW(2, mbar_wait(&tready[ntr % NA], (ntr / NA) & 1));
            ++ntr;
            const uint8_t* rr = sA + s * UNIT + row * 128;
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
              const float4 x = *reinterpret_cast<const float4*>(rr + ((cc ^ (row & 7)) * 16));
              const float* w = sCW + 64 + kc * 32 + cc * 4;
              yv = fmaf(w[0], x.x, yv);
              yv = fmaf(w[1], x.y, yv);
              yv = fmaf(w[2], x.z, yv);
              yv = fmaf(w[3], x.w, yv);
            }
            if (a.discard) discard_line(a.pub + tplane * pub_plane_floats + (ts * TM + row) * 64 + kc * 32);
            named_sync_f(1, 128);
            if (leader) mbar_arrive(&aempty[s]);
          }
        }
        const int64_t l = (int64_t)t * TM + row;
        if (l < a.L) {
          const int64_t o = (int64_t)k.seq * a.L + l;
          a.y[o] = fmaf(dval, __ldg(a.u + o), yv);
        }
      }
      // ---- chunk complete: its loads and discards are done
      named_sync_f(1, 128);
      if (leader) {
        __threadfence();
        atomicAdd(a.done + k.q, 1u);
      }
    }
  }
  if (a.dbg) {
    const int role = warp == 0 ? 0 : warp == 1 ? 1 : warp == STORE_WARP ? 4 : warp >= 6 ? 2 : 3;
    const bool rep = (warp == 0 || warp == 1 || warp == STORE_WARP) ? lane == 0 : (lane == 0 && (warp == 2 || warp == 6));
    if (rep)
      for (int i = 0; i < 4; ++i) atomicAdd(a.dbg + role * 4 + i, dacc[i]);
    if (threadIdx.x == 0) atomicAdd(a.dbg + 20, (unsigned long long)(clock64() - t_start));
  }
#undef TW
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tbase);
}

// ----------------------------------------------------------------------------- Krylov image
// img[s][h][ch][n][e] (h = 0 hi, 1 lo; ch = 0..31; n = 0..63; e = 0..3): the K-major
// no-swizzle shared-memory image of Kr^T (k' = 4 ch + e, lag = 127 - k'), zero for lags >= 2^Kc.
__global__ void kr_image_kernel(const double* Kr, const int* Kc, float* img, int n) {
  const int64_t tot = (int64_t)n * 8192;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = e / 8192;
    const int r = (int)(e % 8192);
    const int ch = r / 256, nn = (r / 4) % 64, ee = r % 4;
    const int lag = 127 - (ch * 4 + ee);
    const double v = (lag < (1 << Kc[s])) ? Kr[(s * 64 + nn) * 128 + lag] : 0.0;
    const float hi = tf32_rna((float)v);
    img[s * 16384 + r] = hi;
    img[s * 16384 + 8192 + r] = tf32_rna((float)(v - (double)hi));
  }
}

int launch_kr_image(const double* Kr, const int* Kc, float* img, int n, cudaStream_t st) {
  const int64_t tot = (int64_t)n * 8192;
  kr_image_kernel<<<(int)std::min<int64_t>(ceil_div(tot, 256), 148 * 8), 256, 0, st>>>(Kr, Kc, img, n);
  CASC_LAUNCHED();
  return CASC_OK;
}

int launch_bank_fused(const BankFusedArg& a, const float* pack_f32, int n_planes_total, int grid, cudaStream_t st) {
  if (a.total_chunks <= 0) return CASC_OK;
  FusedMaps maps;
  memset(&maps, 0, sizeof(maps));
  if (!map3d(&maps.pub, a.pub, true, 64, (int64_t)a.ntiles * TM, (int64_t)a.S * a.NL, TM)) return CASC_ERR_CUDA;
  if (!map3d(&maps.P, pack_f32, true, 64, 64, n_planes_total, 64)) return CASC_ERR_CUDA;
  if (cudaFuncSetAttribute(bank_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES) !=
      cudaSuccess)
    return CASC_ERR_CUDA;
  // CTAs wait on one another (publication flags, sequence-slot counters): a cooperative launch
  // guarantees that every CTA of the grid is resident at once (one per SM here)
  int dev = 0, coop = 0, per_sm = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bank_fused_kernel, THREADS, SMEM_BYTES) != cudaSuccess)
    return CASC_ERR_CUDA;
  if (!coop || grid > per_sm * sms) return CASC_ERR_UNSUPPORTED;
  BankFusedArg arg = a;
  void* params[] = {(void*)&maps, (void*)&arg};
  if (cudaLaunchCooperativeKernel((const void*)bank_fused_kernel, dim3(grid), dim3(THREADS), params, SMEM_BYTES, st) !=
      cudaSuccess) {
    (void)cudaGetLastError();
    return CASC_ERR_CUDA;
  }
  count_launch();
  return CASC_OK;
}

}  // namespace casc
