// Host sequencing of the tensor-core bank path (SISO channels, fp32 mode, m in {16, 32, 64}).
//   derived : Krylov columns Abar^j Bbar (j < 2^Kc) by doubling with the powers
//             [Kr_{2^i + j} = P_i Kr_j], tf32 hi/lo image; w = C P_Ne; fp32 copies of C, D;
//             pair weights Q_k = P_{k+1} P_k (float64 product, tf32 hi/lo planes)
//   head    : v^(Kc) (stages 0..Kc-1 with Bbar u)                     -> Va
//   stages  : k = Kc .. Ne-1, two per pass where possible (R23):
//               v^(k+2) = v + P_k v_{l-2^k} + P_{k+1} v_{l-2^(k+1)} + Q_k v_{l-3*2^k}
//             = (I + P_{k+1} z^-2s)(I + P_k z^-s) v, the product of two adjacent factors of
//             PAPER.md Eq. 5; a last odd stage runs alone.                 Va <-> Vb
//   tail    : stage Ne + y = C v + D u                                 -> y
//             (m = 64: the producer of each channel's last state writes (C v, C P_Ne v) per row
//             instead of v, and the tail adds the shifted parts and D u, R24)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <numeric>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "bank_tc.cuh"
#include "profile.cuh"
#include "engine.cuh"
#include "mimo_tc.cuh"

namespace casc {
cudaEvent_t g_timing_t0 = nullptr;   // CASC_TIMING diagnostics: origin recorded by casc_run_host
// CASC_TIMING diagnostics: labelled events recorded without synchronising, printed by
// engine_bank_pipelined after its final synchronisation
static std::vector<std::pair<std::string, cudaEvent_t>> g_marks;
void timing_mark(const std::string& what, cudaStream_t s) {
  if (!getenv("CASC_TIMING") || !g_timing_t0) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, s);
  g_marks.emplace_back(what, e);
}
void timing_print() {                              // after a device synchronisation
  for (auto& mk : g_marks) {
    float t;
    cudaEventElapsedTime(&t, g_timing_t0, mk.second);
    fprintf(stderr, "casc timing: %8.3f ms  %s\n", t, mk.first.c_str());
    cudaEventDestroy(mk.second);
  }
  g_marks.clear();
}

static constexpr int kHeadK = 7;      // Krylov head covers stages 0..6 (128 lags)
static constexpr int kMetaInts = 5;   // per-channel host table: Neff | Kc | parity | order | iota

// the fused output parts (R24-R26) for m = 64; CASC_BANK_AB=0 stores v and runs the separate tail
// (tests compare the two)
// NEXT-3: skip the zero upper blocks of lower-triangular stage weights (CASC_BANK_TRI=0: dense MMAs;
// the tests compare the two bitwise)
static bool bank_tri_enabled() {
  static const bool on = [] {
    const char* e = getenv("CASC_BANK_TRI");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool bank_ab_enabled() {
  static const bool on = [] {
    const char* e = getenv("CASC_BANK_AB");
    return !(e && e[0] == '0');
  }();
  return on;
}

// stage kernels: m % 64 == 0 runs stage pairs (R23) on the history-resident tensor-core
// kernel (bank_hist.cu; the multi-source TMA GEMM of mimo_tc.cu where it does not apply); m = 16, 32
// run one stage per pass on the CUDA-core register-prefetch kernel (bank_stage_rp.cu: HBM-bound)
static char stage_variant(int m) { return m % 64 == 0 ? 't' : 'r'; }

static int pair_slots(int n_max) { return n_max > kHeadK ? (n_max - kHeadK + 1) / 2 : 0; }

struct BankWs {
  int* meta;      // Neff | Kc | parity | order | iota   (kMetaInts n ints)
  double* Kr64;   // [n][m][128]
  float* krT;     // [n][2][m][128]
  void* kr16;     // m = 64: [n][16][2m][8] fp16 head weights (R33)
  float* kinv;    // m = 64: [n][m] their inverse column scales
  double* w64;    // [n][m]
  float *w32, *c32, *d32;
  float* pvec;   // [n][kMaxParts][m] output-part row vectors (R24-R26)
  double* Q64;    // [n][m][m] scratch for one pair weight
  float* Q32;     // [n][qslots][2][m][m] pair weights, tf32 hi/lo planes
  float* parts;   // [kMaxParts][n * batch * L] fused output parts of the last stages (R24-R26)
  int* tri;       // [n] Abar lower triangular (NEXT-3: the stage kernel skips the zero blocks)
  void *Va, *Vb;
  size_t bytes;
};

static BankWs carve_bank(void* ws, int n, int m, int64_t L, int batch, int qslots) {
  Carver c(ws);
  BankWs w{};
  w.meta = c.take<int>((size_t)kMetaInts * n);
  w.Kr64 = c.take<double>((size_t)n * m * 128);
  w.krT = c.take<float>((size_t)n * 2 * m * 128);
  w.kr16 = c.take<uint16_t>(m == 64 ? (size_t)n * 2 * m * 128 : 0);
  w.kinv = c.take<float>(m == 64 ? (size_t)n * m : 0);
  w.w64 = c.take<double>((size_t)n * m);
  w.w32 = c.take<float>((size_t)n * m);
  w.c32 = c.take<float>((size_t)n * m);
  w.d32 = c.take<float>((size_t)n);
  w.pvec = c.take<float>((size_t)n * kMaxParts * m);
  w.Q64 = c.take<double>(qslots ? (size_t)n * m * m : 0);
  w.Q32 = c.take<float>((size_t)n * qslots * 2 * m * m);
  w.parts = c.take<float>(m == 64 ? (size_t)kMaxParts * n * batch * (size_t)L : 0);
  w.tri = c.take<int>((size_t)n);
  const size_t vbytes = (size_t)n * batch * (size_t)L * m * sizeof(float);
  w.Va = c.take<char>(vbytes);
  w.Vb = c.take<char>(vbytes);
  w.bytes = c.bytes();
  return w;
}

bool bank_tc_path(int m, int p, int q, int mode) {
  static const bool force_simt = [] {
    const char* e = getenv("CASC_FORCE_SIMT");
    return e && e[0] == '1';
  }();
  return !force_simt && p == 1 && q == 1 && mode == CASC_FP32 && bank_tc_supported(m);
}

size_t bank_ws_bytes(int n, int m, int64_t L, int batch, int n_max) {
  return carve_bank(nullptr, n, m, L, batch, stage_variant(m) == 't' ? pair_slots(n_max) : 0).bytes;
}

static int pick_group(int64_t ntiles, int64_t seqs, int want) {
  int g = want;
  while (g > 1 && ceil_div(ntiles, g) * seqs < 2 * 148) g /= 2;
  return g;
}

// Q32[s][slot][h] (tf32 hi / lo plane) from Q64[s] for channels with Neff[s] >= need
__global__ void pair_split_kernel(const double* Q64, float* Q32, const int* Neff, int need, int n, int m,
                                  int qslots, int slot) {
  const int64_t mm = (int64_t)m * m, tot = (int64_t)n * mm;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = e / mm, ij = e % mm;
    if (Neff[s] < need) continue;
    const double x = Q64[e];
    const float hi = tf32_rna((float)x);
    float* base = Q32 + ((s * qslots + slot) * 2) * mm;
    base[ij] = hi;
    base[mm + ij] = tf32_rna((float)(x - (double)hi));
  }
}

// One wave of n channels; Pw points at the wave's first channel inside the full pack.
struct BankStream {        // host-buffer run: output channels copied out as soon as they are final
  void* y_host = nullptr;           // pinned [n][batch][L] (null: no streaming)
  // y_host is device-mapped pinned memory: the wave's last emission (its deepest channels, nothing
  // left to overlap with on the last wave) is stored into it by one copy kernel (a scattered channel
  // list in one launch; one copy per channel run costs ~4 us of copy-engine overhead each: 86
  // scattered channels 0.72 vs 0.44 ms, tools/ubench/zc_d2h.cu). Earlier emissions stay on the copy
  // engine: the copy kernel running beside the stage passes slowed them (E2: 2.94 vs 2.23 ms)
  bool zero_copy = false;
  cudaStream_t cout = nullptr;      // copy-out stream
  std::vector<cudaEvent_t>* events = nullptr;   // created here, destroyed by the caller
  // the wave's input arrives in n_chunks chunks of channels [bounds[i], bounds[i+1]) (memory order),
  // submitted by submit_inputs() after the wave's channel table upload (a host->device copy queues
  // behind every copy submitted before it on the copy engine); the head runs per chunk after
  // u_events[i]
  int n_chunks = 0;
  const int* bounds = nullptr;
  const cudaEvent_t* u_events = nullptr;
  std::function<int()> submit_inputs;
  const int* dmeta = nullptr;        // the wave's channel table, already on the device (no upload)
};
// copies the listed channels' rows (row4 float4 each) from device y to the device-mapped pinned
// host buffer: a handful of CTAs saturate PCIe (tools/ubench/zc_d2h.cu: 8 CTAs 52 GB/s)
constexpr int kEmitCtas = 16;
__global__ void emit_rows_kernel(const float4* __restrict__ src, float4* dst, const int* __restrict__ list,
                                 int n_list, int64_t row4) {
  const int64_t total = (int64_t)n_list * row4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = (int64_t)list[i / row4] * row4 + i % row4;
    dst[o] = src[o];
  }
}
// the per-channel table of a wave (kMetaInts n ints): Neff | Kc | parity of the pass count (which
// buffer holds the final state) | channels by decreasing Neff | identity. Returns max Neff.
static int fill_meta(int n, int m, int64_t L, const int* N_host, int* meta) {
  const char variant = stage_variant(m);
  int *Neff = meta, *Kc = Neff + n, *par = Neff + 2 * n, *order = Neff + 3 * n, *iota = Neff + 4 * n;
  int maxNe = 0;
  for (int s = 0; s < n; ++s) {
    Neff[s] = eff_order(N_host[s], L);
    Kc[s] = std::min(kHeadK, Neff[s]);
    const int nstream = Neff[s] - Kc[s];            // streaming stages of this channel
    par[s] = (variant == 't' ? (nstream + 1) / 2 : nstream) % 2;   // passes -> final buffer
    maxNe = std::max(maxNe, Neff[s]);
  }
  std::iota(order, order + n, 0);
  std::iota(iota, iota + n, 0);
  std::stable_sort(order, order + n, [&](int a, int b) { return Neff[a] > Neff[b]; });
  return maxNe;
}
static int bank_wave(int n, int m, int64_t L, int batch, const int* N_host, int N_max, const PackLayout& Pw,
                     const double* Bbar, const double* C, const double* D, const float* u, float* y, void* ws,
                     size_t ws_bytes, cudaStream_t st, int* pinned_meta = nullptr, const BankStream* bs = nullptr);

// Bounded-memory bank: with a workspace smaller than the whole bank needs, the channels are
// processed in consecutive waves of as many channels as fit (each wave is an independent bank).
int engine_bank_tc(int n, int m, int64_t L, int batch, const int* N_host, int N_max, const void* pack,
                   const double* Bbar, const double* C, const double* D, const void* u, void* y, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  int maxNe = 0;
  for (int s = 0; s < n; ++s) maxNe = std::max(maxNe, eff_order(N_host[s], L));
  const int qslots = stage_variant(m) == 't' ? pair_slots(maxNe) : 0;
  int nw = n;
  while (nw > 0 && carve_bank(nullptr, nw, m, L, batch, qslots).bytes > ws_bytes) {
    const size_t per = carve_bank(nullptr, 1, m, L, batch, qslots).bytes;
    const int guess = (int)std::min<size_t>((size_t)nw - 1, ws_bytes / std::max<size_t>(per, 1));
    nw = guess;
  }
  if (nw < 1) {
    if (getenv("CASC_DEBUG")) fprintf(stderr, "casc: bank wave does not fit: ws=%zu one=%zu\n", ws_bytes, carve_bank(nullptr, 1, m, L, batch, qslots).bytes);
    return CASC_ERR_WORKSPACE;
  }
  PackLayout P = pack_layout(const_cast<void*>(pack), n, m, N_max, CASC_FP32);
  const int64_t slot_mm = (int64_t)(N_max + 1) * m * m;
  for (int c0 = 0; c0 < n; c0 += nw) {
    const int cn = std::min(nw, n - c0);
    PackLayout Pw = P;
    Pw.p64 += c0 * slot_mm;
    Pw.f32 += c0 * slot_mm * 2;
    const int64_t sig = (int64_t)c0 * batch * L;
    const int rc = bank_wave(cn, m, L, batch, N_host + c0, N_max, Pw, Bbar + (int64_t)c0 * m, C + (int64_t)c0 * m,
                             D ? D + c0 : nullptr, static_cast<const float*>(u) + sig, static_cast<float*>(y) + sig,
                             ws, ws_bytes, st);
    if (rc) return rc;
  }
  return CASC_OK;
}

// End to end from host buffers with the transfers overlapped (casc_run_host): per wave, the input
// copy (copy-in stream) overlaps the previous wave's compute, and each group of channels whose
// cascade is complete (the head for Ne <= 7, then every stage pass) gets its tail and its output
// copy (copy-out stream) while the remaining passes run. u_h / y_h should be pinned. The caller
// holds the device context's lock (cascade_api.cu). CASC_ERR_WORKSPACE if not even one channel fits,
// CASC_ERR_UNSUPPORTED for shapes without the fused output parts (the caller then runs the serial
// path).
int engine_bank_pipelined(int n, int m, int64_t L, int batch, const int* N_host, int N_max, const void* pack,
                          const double* Bbar, const double* C, const double* D, float* u_dev, float* y_dev,
                          const void* u_h, const void* y_h, void* ws, size_t ws_bytes, cudaStream_t st,
                          DevCtx* ctx) {
  if (m != 64 || !bank_ab_enabled()) return CASC_ERR_UNSUPPORTED;
  int maxNe = 0;
  for (int s = 0; s < n; ++s) maxNe = std::max(maxNe, eff_order(N_host[s], L));
  const int qslots = pair_slots(maxNe);
  // channels per wave (bounded memory, as engine_bank_tc)
  int nw = n;
  while (nw > 0 && carve_bank(nullptr, nw, m, L, batch, qslots).bytes > ws_bytes) {
    const size_t per = carve_bank(nullptr, 1, m, L, batch, qslots).bytes;
    nw = (int)std::min<size_t>((size_t)nw - 1, ws_bytes / std::max<size_t>(per, 1));
  }
  if (nw < 1) return CASC_ERR_WORKSPACE;
  int rc;
  if ((rc = ctx->ensure_pinned((size_t)kMetaInts * n))) return rc;
  std::vector<cudaEvent_t> events;
  auto new_event = [&](cudaEvent_t* e) -> int {
    CASC_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    events.push_back(*e);
    return CASC_OK;
  };
  // u may be overwritten only after earlier work on st: ctx->inputs_free, recorded by the caller
  // after its parameter copies and before the powers (an input copy submitted ahead of the
  // parameter copies would delay them on the copy engine; round 1 measured that order slower)
  CASC_TRY(cudaStreamWaitEvent(ctx->in, ctx->inputs_free, 0));
  const size_t row = (size_t)batch * L * sizeof(float);
  // wave sizes (CASC_WAVE_RAMP = r, 0: uniform): ramp up from nw/r channels and back down (s, 2s,
  // ..., nw, ..., 2s, s) so the first wave's compute starts early and the last wave's output tail is
  // short; each wave's input copy overlaps the previous wave's compute. Measured (E2 e2e, one box,
  // with 4 input chunks): r = 0 4.58, 4 4.49, 16 5.21 ms; E5 760 ms for all (A/B, tools/ab)
  std::vector<int> wsz;
  static const int ramp_div = [] {
    const char* e = getenv("CASC_WAVE_RAMP");
    return e ? std::max(0, atoi(e)) : 4;
  }();
  const int s0 = ramp_div ? std::max(1, nw / ramp_div) : nw;
  if (ramp_div && n >= 4 * s0 && nw >= 4) {
    std::vector<int> up;
    int total = 0;
    for (int M = s0; M < nw && 2 * (total + M) <= n; M *= 2) { up.push_back(M); total += M; }
    wsz = up;
    for (int rest = n - 2 * total; rest > 0;) { const int t = std::min(nw, rest); wsz.push_back(t); rest -= t; }
    wsz.insert(wsz.end(), up.rbegin(), up.rend());
  } else {
    for (int c0 = 0; c0 < n; c0 += nw) wsz.push_back(std::min(nw, n - c0));
  }
  const int waves = (int)wsz.size();
  std::vector<int> wc0(waves + 1, 0);
  for (int w = 0; w < waves; ++w) wc0[w + 1] = wc0[w] + wsz[w];
  // input chunks per wave (CASC_E2E_CHUNKS): the head runs per chunk as it lands (E2 e2e with the
  // ramp, after the bank pass's walk fix: 1 chunk 4.18, 2 4.09, 4 4.23 ms -- smaller head launches
  // fill the GPU less)
  static const int chunks = [] {
    const char* e = getenv("CASC_E2E_CHUNKS");
    return e ? std::max(1, atoi(e)) : 2;
  }();
  std::vector<std::vector<int>> bounds(waves);
  std::vector<std::vector<cudaEvent_t>> u_ev(waves);
  for (int w = 0; w < waves; ++w) {
    const int nc = std::min(wsz[w], chunks);
    bounds[w].resize(nc + 1);
    u_ev[w].resize(nc);
    for (int i = 0; i <= nc; ++i) bounds[w][i] = (int)((int64_t)wsz[w] * i / nc);
    for (int i = 0; i < nc; ++i)
      if ((rc = new_event(&u_ev[w][i]))) return rc;
  }
  // the input copies of wave w are submitted by the wave itself, after its channel table upload: a
  // small host->device copy queues behind every copy submitted before it on the copy engine, so
  // submitting all waves' inputs up front delayed wave 0 by the whole input (E5: 140 ms); wave
  // w+1's copies still run during wave w's compute
  // every wave's channel table in one upload ahead of the inputs (a table copy on st would queue
  // behind the input copies on the copy engine and hold the head back until the whole input landed)
  if ((rc = ctx->ensure_dmeta((size_t)kMetaInts * n))) return rc;
  // outputs: stored straight into y_h when it is device-mapped pinned memory (else copied out)
  void* y_map = const_cast<void*>(y_h);
  bool zero_copy = false;
  {
    cudaPointerAttributes pa{};
    static const bool zc_off = getenv("CASC_NO_ZERO_COPY") != nullptr;
    if (!zc_off && cudaPointerGetAttributes(&pa, y_h) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
        pa.devicePointer) {
      y_map = pa.devicePointer;
      zero_copy = (batch * L) % 4 == 0 && ((uintptr_t)y_map & 15) == 0;
      if (!zero_copy) y_map = const_cast<void*>(y_h);
    }
    cudaGetLastError();                              // a pageable pointer may leave an error behind
  }
  for (int w = 0; w < waves; ++w) fill_meta(wsz[w], m, L, N_host + wc0[w], ctx->pinned + (size_t)kMetaInts * wc0[w]);
  cudaEvent_t meta_ev;
  if ((rc = new_event(&meta_ev))) return rc;
  CASC_TRY(cudaMemcpyAsync(ctx->dmeta, ctx->pinned, sizeof(int) * kMetaInts * (size_t)n, cudaMemcpyHostToDevice, ctx->in));
  CASC_TRY(cudaEventRecord(meta_ev, ctx->in));
  CASC_TRY(cudaStreamWaitEvent(st, meta_ev, 0));
  PackLayout P = pack_layout(const_cast<void*>(pack), n, m, N_max, CASC_FP32);
  const int64_t slot_mm = (int64_t)(N_max + 1) * m * m;
  for (int w = 0; w < waves && rc == CASC_OK; ++w) {
    const int c0 = wc0[w], cn = wsz[w];
    const size_t off = (size_t)c0 * row;
    BankStream bs;
    bs.y_host = (char*)y_map + off;
    bs.zero_copy = zero_copy && w == waves - 1;
    bs.cout = ctx->out;
    bs.events = &events;
    bs.n_chunks = (int)u_ev[w].size();
    bs.bounds = bounds[w].data();
    bs.u_events = u_ev[w].data();
    bs.dmeta = ctx->dmeta + (size_t)kMetaInts * c0;
    bs.submit_inputs = [&, w, off]() -> int {
      const std::vector<int>& b = bounds[w];
      for (int i = 0; i + 1 < (int)b.size(); ++i) {
        CASC_TRY(cudaMemcpyAsync((char*)u_dev + off + (size_t)b[i] * row, (const char*)u_h + off + (size_t)b[i] * row,
                                 (size_t)(b[i + 1] - b[i]) * row, cudaMemcpyHostToDevice, ctx->in));
        CASC_TRY(cudaEventRecord(u_ev[w][i], ctx->in));
        timing_mark("input chunk " + std::to_string(i), ctx->in);
      }
      timing_mark("input copied, wave " + std::to_string(w), ctx->in);
      return CASC_OK;
    };
    PackLayout Pw = P;
    Pw.p64 += c0 * slot_mm;
    Pw.f32 += c0 * slot_mm * 2;
    const int64_t sig = (int64_t)c0 * batch * L;
    rc = bank_wave(cn, m, L, batch, N_host + c0, N_max, Pw, Bbar + (int64_t)c0 * m, C + (int64_t)c0 * m,
                   D ? D + c0 : nullptr, u_dev + sig, y_dev + sig, ws, ws_bytes, st, ctx->pinned + kMetaInts * (size_t)c0,
                   &bs);
  }
  if (getenv("CASC_TIMING") && g_timing_t0) {       // diagnostics: when each stream finishes
    cudaEvent_t a, b, c;
    cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&c);
    cudaEventRecord(a, ctx->in); cudaEventRecord(b, st); cudaEventRecord(c, ctx->out);
    cudaDeviceSynchronize();
    float ta, tb, tc;
    cudaEventElapsedTime(&ta, g_timing_t0, a); cudaEventElapsedTime(&tb, g_timing_t0, b); cudaEventElapsedTime(&tc, g_timing_t0, c);
    timing_print();
    fprintf(stderr, "casc timing: input copies done %.3f, compute done %.3f, output copies done %.3f ms\n", ta, tb, tc);
    cudaEventDestroy(a); cudaEventDestroy(b); cudaEventDestroy(c);
  }
  // every stream is drained before returning, also on error: no copy into or out of the caller's
  // host buffers is in flight after the call
  cudaError_t e1 = cudaStreamSynchronize(ctx->out), e2 = cudaStreamSynchronize(st);
  cudaError_t e3 = cudaStreamSynchronize(ctx->in);
  for (auto& e : events) cudaEventDestroy(e);
  if (rc) return rc;
  return (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) ? CASC_ERR_CUDA : CASC_OK;
}

// pinned_meta: optional pinned host staging for the channel table (6n ints, untouched until the
// stream has consumed it), so the upload is a true asynchronous copy
static int bank_wave(int n, int m, int64_t L, int batch, const int* N_host, int N_max, const PackLayout& Pw,
                     const double* Bbar, const double* C, const double* D, const float* u, float* y, void* ws,
                     size_t ws_bytes, cudaStream_t st, int* pinned_meta, const BankStream* bs) {
  const char variant = stage_variant(m);
  // output fusion: the producer of each channel's last state writes (C v, C P_Ne v) instead of
  // v (R24); taken with the m = 64 tensor-core stage kernels and head
  const bool use_ab = m == 64 && bank_ab_enabled();
  // with a pre-uploaded table (bs->dmeta) the host copy is rebuilt locally (the pinned staging may
  // still be in flight)
  const bool pre = bs && bs->dmeta;
  std::vector<int> meta_v((pinned_meta && !pre) ? 0 : (size_t)kMetaInts * n);
  int* meta = (pinned_meta && !pre) ? pinned_meta : meta_v.data();
  int *Neff = meta, *Kc = Neff + n, *order = Neff + 3 * n;
  const int maxNe = fill_meta(n, m, L, N_host, meta);
  const int qslots = variant == 't' ? pair_slots(maxNe) : 0;
  BankWs w = carve_bank(ws, n, m, L, batch, qslots);
  if (ws_bytes < w.bytes) {
    if (getenv("CASC_DEBUG")) fprintf(stderr, "casc: bank wave ws=%zu need=%zu n=%d\n", ws_bytes, w.bytes, n);
    return CASC_ERR_WORKSPACE;
  }
  const PackLayout& P = Pw;
  const int64_t mm = (int64_t)m * m;
  int rc;
  // R24-R26 (common.cuh OutParts): y is formed from parts written by the kernel producing
  // v^(Ne-d); with fold, d = 1 for an odd number of streaming stages (no single-stage pass) and
  // d = 2 for an even number >= 2 (the last stage-pair pass is skipped). Planned only where every
  // pass producing d > 0 parts runs on the history-resident kernel (or is the head).
  // CASC_BANK_FOLD = 1 (R25, default) | 0 (R24 only: every streaming stage runs; the tests compare
  // the two regroupings). R26 (fold 2: also skip the last stage-pair pass) measured slower (E2 3.90
  // vs 3.75 ms, E5 807 vs 768 ms: eight-part epilogues cost more than the skipped passes save).
  static const int fold_mode = [] {
    const char* e = getenv("CASC_BANK_FOLD");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  int fold = (use_ab && variant == 't') ? fold_mode : 0;
  for (int c = 0; fold && c < n; ++c) {
    const int d = fold_depth(Neff[c], Kc[c], fold), lp = Neff[c] - d;
    if (d > 0 && lp > Kc[c] && !bank_hist_ok(L, (int64_t)1 << (lp - 2), 3, 0)) fold = 0;
  }
  std::vector<int> Lp(n);                          // the state level each channel's parts come from
  for (int c = 0; c < n; ++c) Lp[c] = Neff[c] - fold_depth(Neff[c], Kc[c], fold);
  if (!pre) CASC_TRY(cudaMemcpyAsync(w.meta, meta, (size_t)kMetaInts * n * sizeof(int), cudaMemcpyHostToDevice, st));
  const int* dm = pre ? bs->dmeta : w.meta;
  const int *dNeff = dm, *dKc = dm + n, *dpar = dm + 2 * n, *dorder = dm + 3 * n, *diota = dm + 4 * n;
  if (bs && bs->submit_inputs && (rc = bs->submit_inputs())) return rc;
  auto count_ge = [&](int need) {                    // channels with Neff >= need: a prefix of order
    int c = 0;
    while (c < n && Neff[order[c]] >= need) ++c;
    return c;
  };
  auto count_lp_ge = [&](int need) {                 // channels with Lp >= need: a prefix of order too
    int c = 0;
    while (c < n && Lp[order[c]] >= need) ++c;
    return c;
  };
  const int64_t plane = (int64_t)n * batch * L;
  OutParts op;
  if (use_ab) {
    op.planes = w.parts; op.plane = plane; op.vec = w.pvec; op.neff = dNeff; op.kc = dKc; op.fold = fold;
  }

  cudaStream_t qs = st;                            // pair weights' stream (side stream below)
  cudaEvent_t q_start = nullptr, q_done = nullptr;
  struct EvGuard {                                 // destroyed once the waits are enqueued
    cudaEvent_t* a; cudaEvent_t* b;
    ~EvGuard() { if (*a) cudaEventDestroy(*a); if (*b) cudaEventDestroy(*b); }
  } ev_guard{&q_start, &q_done};
  // ---- derived: Krylov columns, w = C P_Ne, fp32 copies, pair weights
  {
    // the pair weights Q_k need only the powers: they run on a side stream under derived + head
    DevCtx* ctx = dev_ctx();
    if (!ctx) return CASC_ERR_CUDA;
    qs = ctx->side;
    CASC_TRY(cudaEventCreateWithFlags(&q_start, cudaEventDisableTiming));
    CASC_TRY(cudaEventCreateWithFlags(&q_done, cudaEventDisableTiming));
    CASC_TRY(cudaEventRecord(q_start, st));
    CASC_TRY(cudaStreamWaitEvent(qs, q_start, 0));
    ProfScope ps(st, K_DERIVED, 0.0, 2.0 * n * (double)m * m * 128);
    if ((rc = launch_bank_derived(P.p64, N_max + 1, Bbar, C, D, dNeff, dKc, w.Kr64, w.krT, w.w64, w.w32, w.c32,
                                  w.d32, use_ab ? w.pvec : nullptr, w.tri, fold, n, m, st, w.kr16, w.kinv)))
      return rc;
    for (int j = 0; j < qslots; ++j) {          // Q_k = P_{k+1} P_k for pass j (k = 7 + 2j)
      const int k = kHeadK + 2 * j;
      if (count_lp_ge(k + 2) == 0) continue;
      DgemmArg q{};
      q.M = m; q.N = m; q.K = m;
      q.A = P.p64 + (k + 1) * mm; q.lda = m; q.sA = (int64_t)(N_max + 1) * mm;
      q.B = P.p64 + k * mm; q.ldb = m; q.sB = (int64_t)(N_max + 1) * mm;
      q.C = w.Q64; q.ldc = m; q.sC = mm;
      q.skip_below = dNeff; q.level = k + 2;
      if ((rc = launch_dgemm(q, n, qs))) return rc;
      pair_split_kernel<<<(int)std::min<int64_t>(ceil_div((int64_t)n * mm, 256), 148 * 8), 256, 0, qs>>>(
          w.Q64, w.Q32, dNeff, k + 2, n, m, qslots, j);
      CASC_LAUNCHED();
    }
    CASC_TRY(cudaEventRecord(q_done, qs));
  }
  const int64_t ntiles = ceil_div(L, 128);
  // streaming outputs (host-buffer run): channels order[a, b) are final -> tail + copy out
  const bool streaming = bs && bs->y_host && use_ab;
  auto emit = [&](int a0, int b0) -> int {
    const int* dlist = dorder + a0;
    const int* hlist = order + a0;
    const int cnt = b0 - a0;
    if (!streaming || cnt <= 0) return CASC_OK;
    BankAbTailArg t{};
    t.op = op; t.u = static_cast<const float*>(u); t.y = static_cast<float*>(y);
    t.d = w.d32; t.n_ch = n; t.L = L; t.batch = batch;
    t.list = dlist; t.n_list = cnt;
    int rc2;
    {
      ProfScope ps(st, K_BANK_TAIL, (double)cnt * batch * L * 24.0, (double)cnt * batch * L * 3);
      if ((rc2 = launch_bank_ab_tail(t, st))) return rc2;
    }
    cudaEvent_t ev;
    CASC_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    bs->events->push_back(ev);
    CASC_TRY(cudaEventRecord(ev, st));
    CASC_TRY(cudaStreamWaitEvent(bs->cout, ev, 0));
    const size_t row = (size_t)batch * L * sizeof(float);
    timing_mark("tail launched for " + std::to_string(cnt) + " channels", st);
    if (bs->zero_copy && a0 == 0) {
      const int64_t row4 = (int64_t)batch * L / 4;
      emit_rows_kernel<<<kEmitCtas, 512, 0, bs->cout>>>(reinterpret_cast<const float4*>(y),
                                                        reinterpret_cast<float4*>(bs->y_host), dlist, cnt, row4);
      CASC_LAUNCHED();
      return CASC_OK;
    }
    for (int i = 0; i < cnt;) {                   // merge runs of consecutive channel ids
      int j = i + 1;
      while (j < cnt && hlist[j] == hlist[j - 1] + 1) ++j;
      CASC_TRY(cudaMemcpyAsync((char*)bs->y_host + (size_t)hlist[i] * row, (const char*)y + (size_t)hlist[i] * row,
                               (size_t)(j - i) * row, cudaMemcpyDeviceToHost, bs->cout));
      i = j;
    }
    return CASC_OK;
  };
  // ---- head: stages 0..Kc-1 (+ Bbar u), all channels
  // the input of a host-buffer run arrives in chunks on a copy stream: the head runs per chunk after
  // it landed (and the D u tails, later on st, after all of them)
  const bool chunked = bs && bs->n_chunks > 0;
  for (int ci = 0; ci < (chunked ? bs->n_chunks : 1); ++ci) {
    if (ci == 0) timing_mark("before head", st);
    if (chunked) CASC_TRY(cudaStreamWaitEvent(st, bs->u_events[ci], 0));
    const int hc0 = chunked ? bs->bounds[ci] : 0, hcn = chunked ? bs->bounds[ci + 1] - hc0 : n;
    BankHeadArg a{};
    a.u = static_cast<const float*>(u); a.krT = w.krT; a.kr16 = static_cast<const __half*>(w.kr16); a.kinv = w.kinv; a.V = static_cast<float*>(w.Va);
    a.sys_list = chunked ? diota + hc0 : dorder; a.n_list = hcn; a.L = L; a.batch = batch;
    if (use_ab) a.op = op;
    ProfScope ps(st, K_BANK_HEAD, (double)hcn * batch * L * (1 + m) * 4.0,
                 (double)hcn * batch * L * 2.0 * m * 128);
    // executed: m = 64 issues three fp16 products per K step (hi.[hi|lo] at N = 128, lo.hi) on the
    // kind::f16 pipe (the bf16 rate)
    if (m == 64) ps.exec((double)hcn * batch * L * (1 + m) * 4.0, 3.0 * hcn * batch * L * 2.0 * m * 128, PIPE_BF16);
    // m = 64: warp-specialized TMA-store head (bank_head_ws.cu); m = 16, 32: CUDA-core head.
    // Measured alternatives not kept: a TMEM-operand variant (1.67 vs 1.30 ms on E2),
    // the head on CTA pairs (same 1.16 ms: the head is bound by the tensor pipe, 69% active)
    if (m == 64) {
      a.tiles_per_cta = pick_group(ntiles, (int64_t)hcn * batch, 64);
      rc = launch_bank_head_ws(m, a, (int64_t)n * batch, st);   // V map: every sequence of the wave
    } else {
      a.tiles_per_cta = pick_group(ntiles, (int64_t)hcn * batch, 16);
      rc = launch_bank_head(m, a, st);
    }
    if (rc) return rc;
    timing_mark("head chunk " + std::to_string(ci), st);
  }
  // cascades whose output parts come from the head (Ne <= 7; with fold also Ne = 8)
  if ((rc = emit(count_lp_ge(kHeadK + 1), n))) return rc;
  auto tmark = [&](const char* what) { timing_mark(std::string(what) + " n=" + std::to_string(n), st); };
  tmark("head done");
  if (q_done) CASC_TRY(cudaStreamWaitEvent(st, q_done, 0));   // the pair weights
  // ---- streaming stages k >= kHeadK over the channels with Neff > k (prefixes of `order`)
  int pass = 0;
  for (int k = kHeadK; k < maxNe; k += (variant == 't' ? 2 : 1), ++pass) {
    const float* Vs = static_cast<const float*>(pass % 2 == 0 ? w.Va : w.Vb);
    float* Vd = static_cast<float*>(pass % 2 == 0 ? w.Vb : w.Va);
    if (variant != 't') {
      const int cnt = count_ge(k + 1);
      BankStageArg a{};
      a.Vs = Vs; a.Vd = Vd; a.P = P.f32; a.k = k; a.slots = N_max + 1;
      a.copy_from = (k == kHeadK) ? 0 : ((int64_t)1 << (k - 1));
      a.sys_list = dorder; a.n_list = cnt; a.L = L; a.batch = batch;
      a.tiles_per_cta = pick_group(ntiles, (int64_t)cnt * batch, 8);
      ProfScope ps(st, K_BANK_STAGE, 2.0 * cnt * batch * L * m * 4.0, 2.0 * cnt * batch * L * (double)mm);
      rc = launch_bank_stage_rp(m, a, st);
      if (rc) return rc;
      continue;
    }
    // pass: stages k and k+1 for channels with Neff >= k+2; stage k alone for Neff == k+1.
    // The destination holds v^(k-2) (two passes ago), equal to v^(k+2) on rows < 2^(k-2).
    const int cnt2 = count_lp_ge(k + 2), cnt1 = count_lp_ge(k + 1) - cnt2;   // cnt1 = 0 with fold
    const int t_first = pass == 0 ? 0 : (int)(((int64_t)1 << (k - 2)) / 128);
    const int64_t planes = (int64_t)n * (N_max + 1) * 2;
    if (cnt2 > 0) {
      MimoGemm g{};
      g.src[0].A = Vs; g.src[0].W = P.f32; g.src[0].K = m; g.src[0].shift = (int64_t)1 << k;
      g.src[0].w_plane_off = 2 * k; g.src[0].w_planes = planes; g.src[0].w_plane_stride = 2 * (N_max + 1);
      g.src[1] = g.src[0];
      g.src[1].shift = (int64_t)2 << k; g.src[1].w_plane_off = 2 * (k + 1);
      g.src[2].A = Vs; g.src[2].W = w.Q32; g.src[2].K = m; g.src[2].shift = (int64_t)3 << k;
      g.src[2].w_plane_off = 2 * pass; g.src[2].w_planes = (int64_t)n * qslots * 2;
      g.src[2].w_plane_stride = 2 * qslots;
      g.n_src = 3; g.R = Vs; g.out = Vd; g.n_out = m; g.L = L; g.batch = batch;
      g.sys_list = dorder; g.n_list = cnt2; g.n_sys_total = n; g.t_first = t_first; g.w_resident = 1;
      if (use_ab) {                                 // channels whose parts come from this pass (Lp == k + 2)
        g.ab_neff = dNeff; g.ab_level = k + 2; g.ab_c = w.c32; g.ab_w = w.w32; g.ab = w.parts; g.ab_plane = plane;
        g.parts = op; g.parts.level = k + 2;
        for (int c = 0; c < n; ++c) g.parts_deep |= (Lp[c] == k + 2 && Lp[c] != Neff[c]);
        if (count_lp_ge(k + 2) > count_lp_ge(k + 3)) g.t_first = 0;   // their parts need every row
      }
      // bytes of the schedule run (SURVEY 8d B_fused): one read + one write of the state for the two
      // stages this pass applies; flops of both stages (bench.py derives the unfused B_ns from them)
      ProfScope ps(st, K_BANK_STAGE, 2.0 * cnt2 * batch * L * m * 4.0, 4.0 * cnt2 * batch * L * (double)mm);
      // executed: three sources x three tf32 products (3xTF32) per row, dense; the history kernel
      // counts what it actually issues (zero blocks of triangular weights skipped, NEXT-3)
      ps.exec(2.0 * cnt2 * batch * L * m * 4.0, 9.0 * 2.0 * cnt2 * batch * L * (double)mm, PIPE_TF32);
      g.tri = bank_tri_enabled() ? w.tri : nullptr;
      g.flop_counter = ps.device_flops();
      rc = launch_bank_hist(g, st);
      if (rc == CASC_ERR_UNSUPPORTED) {
        ps.drop_device_flops();
        rc = launch_mimo_gemm(g, true, st);
      }
      if (rc) return rc;
    }
    if (cnt1 > 0) {                                // single stage k for Ne == k + 1 (none with fold)
      MimoGemm g{};
      g.src[0].A = Vs; g.src[0].W = P.f32; g.src[0].K = m; g.src[0].shift = (int64_t)1 << k;
      g.src[0].w_plane_off = 2 * k; g.src[0].w_planes = planes; g.src[0].w_plane_stride = 2 * (N_max + 1);
      g.n_src = 1; g.R = Vs; g.out = Vd; g.n_out = m; g.L = L; g.batch = batch;
      g.sys_list = dorder + cnt2; g.n_list = cnt1; g.n_sys_total = n; g.t_first = t_first;
      if (use_ab) {                                 // every channel here ends with stage k
        g.ab_neff = dNeff; g.ab_level = k + 1; g.ab_c = w.c32; g.ab_w = w.w32; g.ab = w.parts; g.ab_plane = plane;
        g.parts = op; g.parts.level = k + 1;
        g.t_first = 0;
      }
      ProfScope ps(st, K_BANK_STAGE, 2.0 * cnt1 * batch * L * m * 4.0, 2.0 * cnt1 * batch * L * (double)mm);
      ps.exec(2.0 * cnt1 * batch * L * m * 4.0, 3.0 * 2.0 * cnt1 * batch * L * (double)mm, PIPE_TF32);
      g.tri = bank_tri_enabled() ? w.tri : nullptr;
      g.flop_counter = ps.device_flops();
      rc = launch_bank_hist(g, st);
      if (rc == CASC_ERR_UNSUPPORTED) {
        ps.drop_device_flops();
        rc = launch_mimo_gemm(g, true, st);
      }
      if (rc) return rc;
    }
    if ((rc = emit(count_lp_ge(k + 3), count_lp_ge(k + 1)))) return rc;   // channels with Lp in {k + 1, k + 2}
  }
  tmark("passes done");
  if (streaming) return CASC_OK;                      // every channel was emitted
  // ---- tail: stage Ne + y = C v + D u
  if (use_ab) {                                     // from the fused (C v, C P_Ne v) parts
    BankAbTailArg a{};
    a.op = op; a.u = static_cast<const float*>(u); a.y = static_cast<float*>(y);
    a.d = w.d32; a.n_ch = n; a.L = L; a.batch = batch;
    ProfScope ps(st, K_BANK_TAIL, (double)n * batch * L * (8 + 8 + 4 + 4), (double)n * batch * L * 3);
    return launch_bank_ab_tail(a, st);
  }
  {
    BankTailArg a{};
    a.Va = static_cast<const float*>(w.Va); a.Vb = static_cast<const float*>(w.Vb); a.parity = dpar;
    a.cvec = w.c32; a.wvec = w.w32; a.d = w.d32; a.Neff = dNeff;
    a.u = static_cast<const float*>(u); a.y = static_cast<float*>(y);
    a.n_ch = n; a.L = L; a.batch = batch;
    ProfScope ps(st, K_BANK_TAIL, (double)n * batch * L * (m + 2) * 4.0, (double)n * batch * L * (4.0 * m + 2));
    if ((rc = launch_bank_tail(m, a, st))) return rc;
  }
  return CASC_OK;
}

}  // namespace casc
