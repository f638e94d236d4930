// Thin inline-PTX helpers for the sm_100a tensor-core path (tcgen05 / TMEM / mbarrier / TMA).
// Descriptor bit layouts follow the PTX ISA "Matrix descriptor" and "Instruction descriptor"
// tables for tcgen05 (the same fields CUTLASS names in cute/arch/mma_sm100_desc.hpp).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace casc {
namespace sm100 {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// The lanes that entered together leave together: lanes spinning independently can exit the
// loop in different iterations, and a .sync.aligned tcgen05.ld / st right after a diverged exit
// corrupted one 32-lane quadrant of a tile in bank_hist.cu (found under load, tools/hist_diag.py).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const unsigned lanes = __activemask();
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
  __syncwarp(lanes);
}

// Whole-warp wait with a warp-uniform exit (vote): code after it stays uniform control flow, so
// ptxas can keep loop-carried MMA operands in uniform registers.
__device__ __forceinline__ void mbar_wait_u(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "vote.sync.all.pred p, p, 0xffffffff;\n\t"
      "@!p bra.uni WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// ------------------------------------------------------------------ proxies / fences
__device__ __forceinline__ void fence_async_smem() {       // generic-proxy smem writes -> async proxy
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// ------------------------------------------------------------------ TMEM
template <int kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {   // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               ::"r"(smem_u32(dst_smem)), "n"(kCols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {      // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}

// 32 lanes x 32-bit, 16 consecutive columns per thread (thread i of the warp <-> lane base+i)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// ------------------------------------------------------------------ UMMA descriptors
// Shared-memory matrix descriptor (64-bit): start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version=1 [46,48) (sm_100), base offset [49,52), lbo mode [52], layout type [61,64).
enum : uint32_t { LAYOUT_NONE = 0, LAYOUT_SW128 = 2, LAYOUT_SW64 = 4, LAYOUT_SW32 = 6 };
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

// Instruction descriptor for kind::tf32 / kind::f16 (32-bit):
// c_format [4,6) (1 = f32), a_format [7,10), b_format [10,13) (f16 = 0, bf16 = 1, tf32 = 2),
// a_major [15], b_major [16] (0 = K-major), N>>3 [17,23), M>>4 [24,29).
enum : uint32_t { FMT_F16 = 0, FMT_BF16 = 1, FMT_TF32 = 2 };
__host__ __device__ constexpr uint32_t make_idesc(uint32_t ab_fmt, int M, int N) {
  return (1u << 4) | (ab_fmt << 7) | (ab_fmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// Warp-collective issue: the whole converged warp executes these and one lane (elect.sync)
// issues. The operands stay warp-uniform, so ptxas keeps them in uniform registers; issuing from
// a single divergent lane instead wraps every MMA in a per-lane waterfall loop with R2UR
// conversions (measured ~95 cycles per MMA vs the 32-cycle floor of an N=64 tf32 MMA).
__device__ __forceinline__ void mma_tf32_w(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_f16_w(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// The 12-MMA form of the chunk below (tools/ubench/ubench_tc.cu measures both): in ONE asm block:
//   d  (+)= A_hi W_hi        dc (+)= A_lo W_hi + A_hi W_lo
// ah/al: TMEM column addresses of the chunk's hi / lo parts (8 columns per K-step); wd/wl: SW128
// K-major descriptors of W hi / lo (32 B per K-step = +2 in the start field). `acc` = 0 starts both
// accumulators. Passing the base operands once lets ptxas form the twelve MMAs' operands with
// uniform-register adds instead of converting every operand per MMA (R2UR), which dominated the
// issue time of the per-MMA helpers.
__device__ __forceinline__ void mma_3xtf32_ts_chunk_w(uint32_t d, uint32_t dc, uint32_t ah, uint32_t al, uint64_t wd,
                                                      uint64_t wl, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 a1, a2, a3, l1, l2, l3;\n\t.reg .b64 w1, w2, w3, v1, v2, v3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %7, 0;\n\t"
      "add.u32 a1, %2, 8;\n\tadd.u32 a2, %2, 16;\n\tadd.u32 a3, %2, 24;\n\t"
      "add.u32 l1, %3, 8;\n\tadd.u32 l2, %3, 16;\n\tadd.u32 l3, %3, 24;\n\t"
      "add.u64 w1, %4, 2;\n\tadd.u64 w2, %4, 4;\n\tadd.u64 w3, %4, 6;\n\t"
      "add.u64 v1, %5, 2;\n\tadd.u64 v2, %5, 4;\n\tadd.u64 v3, %5, 6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %4, %6, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [%3], %4, %6, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [%2], %5, %6, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a1], w1, %6, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [l1], w1, %6, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [a1], v1, %6, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a2], w2, %6, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [l2], w2, %6, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [a2], v2, %6, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a3], w3, %6, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [l3], w3, %6, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [a3], v3, %6, 1;\n\t}"
      ::"r"(d), "r"(dc), "r"(ah), "r"(al), "l"(wd), "l"(wl), "r"(idesc), "r"(acc));
}
// One K chunk (32 tf32 = 4 K-steps) of the 3xTF32 product with A in TMEM (ah / al: TMEM columns of
// the chunk's hi / lo parts, 8 columns per K-step; wd: SW128 K-major descriptor of [W hi | W lo],
// 32 B per K-step = +2 in the start field), in ONE asm block so ptxas forms the operands with
// uniform-register adds. The hi.hi and hi.lo products share A = a_hi, so one N = 2*64 MMA
// against [W hi | W lo] (lo stored right after hi: one K-major SW128 operand of 128 rows) writes
// hi.hi to d and hi.lo to d + 64 = dc; lo.hi then accumulates into dc. Fewer MMA instructions and
// operands per chunk (the issuing warp's instruction stream bounds the N = 64 bank stage).
__device__ __forceinline__ void mma_3xtf32_ts_chunk8_w(uint32_t d, uint32_t dc, uint32_t ah, uint32_t al,
                                                       uint64_t wd, uint32_t idesc128, uint32_t idesc64,
                                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 a1, a2, a3, l1, l2, l3;\n\t.reg .b64 w1, w2, w3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %6, 0;\n\t"
      "add.u32 a1, %2, 8;\n\tadd.u32 a2, %2, 16;\n\tadd.u32 a3, %2, 24;\n\t"
      "add.u32 l1, %3, 8;\n\tadd.u32 l2, %3, 16;\n\tadd.u32 l3, %3, 24;\n\t"
      "add.u64 w1, %4, 2;\n\tadd.u64 w2, %4, 4;\n\tadd.u64 w3, %4, 6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %4, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [%3], %4, %7, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a1], w1, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [l1], w1, %7, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a2], w2, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [l2], w2, %7, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a3], w3, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [l3], w3, %7, 1;\n\t}"
      ::"r"(d), "r"(dc), "r"(ah), "r"(al), "l"(wd), "r"(idesc128), "r"(acc), "r"(idesc64));
}
// The same chunk for a LOWER-TRIANGULAR weight W (W[n][k] = 0 for k > n: powers of a lower-
// triangular Abar, "structured representation"). K-step t of the
// 64 x 64 product (k in [8t, 8t + 8), t = 4 KC + i) meets only rows n >= 8t of W, so each MMA starts
// at row n0 = 16 floor(t / 2) (UMMA N granularity 16): the B descriptor moves down n0 rows (n0 * 128
// B: whole 1024-B SW128 atoms), the accumulator columns move right by n0 and N shrinks by n0
//   hi.[W hi | W lo]: rows n0 .. 127 of the stacked operand (N = 128 - n0) into d + n0 (the hi.lo
//                     half keeps all 64 rows: its zero rows are computed, not skipped)
//   lo.W hi:          rows n0 .. 63 (N = 64 - n0) into dc + n0.
// The skipped products are exact zeros, so every accumulator column receives the same non-zero
// terms in the same order as the dense chunk. The first MMA of a tile has t = 0 (n0 = 0) and still
// initialises all 128 columns. Issued work per chunk: sum_i (192 - 2 n0_i) / (4 * 192) of dense.
template <int KC>
__device__ __forceinline__ void mma_3xtf32_ts_chunk8_tri_w(uint32_t d, uint32_t dc, uint32_t ah, uint32_t al,
                                                           uint64_t wd, uint32_t acc) {
  constexpr uint32_t n0a = 32 * KC, n0b = 32 * KC + 16;                   // K-steps 0-1 / 2-3
  constexpr uint32_t i128a = make_idesc(FMT_TF32, 128, 128 - n0a), i64a = make_idesc(FMT_TF32, 128, 64 - n0a);
  constexpr uint32_t i128b = make_idesc(FMT_TF32, 128, 128 - n0b), i64b = make_idesc(FMT_TF32, 128, 64 - n0b);
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 d0, d1, c0, c1, a1, a2, a3, l1, l2, l3;\n\t.reg .b64 w0, w1, w2, w3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\t"
      "add.u32 d0, %0, %6;\n\tadd.u32 d1, %0, %7;\n\tadd.u32 c0, %1, %6;\n\tadd.u32 c1, %1, %7;\n\t"
      "add.u32 a1, %2, 8;\n\tadd.u32 a2, %2, 16;\n\tadd.u32 a3, %2, 24;\n\t"
      "add.u32 l1, %3, 8;\n\tadd.u32 l2, %3, 16;\n\tadd.u32 l3, %3, 24;\n\t"
      "add.u64 w0, %4, %8;\n\tadd.u64 w1, %4, %9;\n\tadd.u64 w2, %4, %10;\n\tadd.u64 w3, %4, %11;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d0], [%2], w0, %12, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [c0], [%3], w0, %13, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d0], [a1], w1, %12, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [c0], [l1], w1, %13, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d1], [a2], w2, %14, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [c1], [l2], w2, %15, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [d1], [a3], w3, %14, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [c1], [l3], w3, %15, 1;\n\t}"
      ::"r"(d), "r"(dc), "r"(ah), "r"(al), "l"(wd), "r"(acc), "n"(n0a), "n"(n0b),
        "n"(n0a * 8 + 0), "n"(n0a * 8 + 2), "n"(n0b * 8 + 4), "n"(n0b * 8 + 6),
        "n"(i128a), "n"(i64a), "n"(i128b), "n"(i64b));
}
// MMA work of one triangular chunk relative to the dense chunk8 (in units of N-columns x K-steps)
template <int KC>
__host__ __device__ constexpr uint32_t tri_chunk_cols() {
  return 2 * ((128 - 32 * KC) + (64 - 32 * KC)) + 2 * ((128 - 32 * KC - 16) + (64 - 32 * KC - 16));
}
__device__ __forceinline__ void mma_commit_w(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
               ::"r"(smem_u32(bar)) : "memory");
}
// Descriptor start-address field holds addr >> 4: a byte offset b (16-B multiple, no carry out of
// the 14-bit field) is added as b >> 4.
__device__ __forceinline__ uint64_t sdesc_add(uint64_t d, uint32_t bytes) { return d + (bytes >> 4); }

// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar)) : "memory");
}

}  // namespace sm100
}  // namespace casc
