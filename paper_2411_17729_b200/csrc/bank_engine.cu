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
#include <numeric>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "bank_tc.cuh"
#include "profile.cuh"
#include "engine.cuh"
#include "mimo_tc.cuh"

namespace casc {
cudaEvent_t g_timing_t0 = nullptr;   // CASC_TIMING diagnostics: origin recorded by casc_run_host

static constexpr int kHeadK = 7;      // Krylov head covers stages 0..6 (128 lags)

// stage-kernel variant (CASC_BANK_STAGE, for A/B measurements), m % 64 == 0:
//   't' (default) stage pairs (R23): one pass applies two adjacent factors of Eq. 5 through a
//       3-source TMA GEMM with the A operands in TMEM and the three weight pairs resident in
//       shared memory; half the HBM passes of 's' (E2: 3.97 vs 4.30 ms for the streaming stages)
//   's' one stage per pass (HBM-bound, ~84% of the measured copy bandwidth)
//   'r' register-prefetch kernel, 'w' warp-specialized CUDA-core variant (m = 16, 32 use 'r')
static char stage_variant(int m) {
  static const char env = [] {
    const char* e = getenv("CASC_BANK_STAGE");
    return e ? e[0] : 't';
  }();
  if (env == 'w' || env == 'r') return env;
  if (m % 64 != 0) return 'r';
  return env == 's' ? 's' : 't';
}

static int pair_slots(int n_max) { return n_max > kHeadK ? (n_max - kHeadK + 1) / 2 : 0; }

// Weight-resident GEMM mode for the stage (CASC_BANK_WRES=1). Measured slower on E2 (5.2 ms vs
// 4.5 ms per step for the stages): the single weight buffer needs a pipeline drain at every
// channel change, which costs more than the ring traffic it saves. Off by default.
static int resident_weights() {
  static const int on = [] {
    const char* e = getenv("CASC_BANK_WRES");
    return e && e[0] == '1' ? 1 : 0;
  }();
  return on;
}

// Weight-resident GEMM for stage pairs (three weight pairs per tile, 96 KB): on by default,
// CASC_BANK_PAIR_WRES=0 reloads the weights per tile through the ring.
static int pair_wres() {
  static const int on = [] {
    const char* e = getenv("CASC_BANK_PAIR_WRES");
    return e && e[0] == '0' ? 0 : 1;
  }();
  return on;
}

struct BankWs {
  int* meta;      // Neff | Kc | parity | order | iota | head-enders by input chunk   (6 n ints)
  double* Kr64;   // [n][m][128]
  float* krT;     // [n][2][m][128]
  double* w64;    // [n][m]
  float *w32, *c32, *d32;
  float* pvec;   // [n][kMaxParts][m] output-part row vectors (R24-R26)
  double* Q64;    // [n][m][m] scratch for one pair weight
  float* Q32;     // [n][qslots][2][m][m] pair weights, tf32 hi/lo planes
  float* parts;   // [kMaxParts][n * batch * L] fused output parts of the last stages (R24-R26)
  void *Va, *Vb;
  size_t bytes;
};

static BankWs carve_bank(void* ws, int n, int m, int64_t L, int batch, int qslots) {
  Carver c(ws);
  BankWs w{};
  w.meta = c.take<int>((size_t)6 * n);
  w.Kr64 = c.take<double>((size_t)n * m * 128);
  w.krT = c.take<float>((size_t)n * 2 * m * 128);
  w.w64 = c.take<double>((size_t)n * m);
  w.w32 = c.take<float>((size_t)n * m);
  w.c32 = c.take<float>((size_t)n * m);
  w.d32 = c.take<float>((size_t)n);
  w.pvec = c.take<float>((size_t)n * kMaxParts * m);
  w.Q64 = c.take<double>(qslots ? (size_t)n * m * m : 0);
  w.Q32 = c.take<float>((size_t)n * qslots * 2 * m * m);
  w.parts = c.take<float>(m == 64 ? (size_t)kMaxParts * n * batch * (size_t)L : 0);
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

static int eff_order_b(int N, int64_t L) {
  if (L <= 2) return 0;
  int kstar = 0;
  while (((int64_t)1 << (kstar + 1)) < L) ++kstar;
  return N < kstar ? N : kstar;
}

// ---------------------------------------------------------------- fused persistent path
// bank_fused.cu: one launch for the whole bank, states in TMEM, levels exchanged through L2.
// Opt-in (CASC_BANK_FUSED=1, read per call) for m = 64 when every channel has Ne >= 7: it is
// correct (tests/test_gpu_bank_fused.py) but measured slower than the multi-kernel path on E2
// (8.9 vs 6.4 ms for head + stages + tail): its tf32 N=64 MMAs are shared-memory-bound (48 cyc
// each, 128 B/cyc) and the per-tile publication chain adds latency; see DESIGN.md.
static bool fused_enabled() {
  const char* e = getenv("CASC_BANK_FUSED");
  return e && e[0] == '1';
}
static bool discard_enabled() {
  static const bool on = [] {
    const char* e = getenv("CASC_DISCARD");
    return !(e && e[0] == '0');
  }();
  return on;
}
static constexpr int kFusedT = 4;           // tiles per chunk (TMEM: 4 x 64 state columns)

struct FusedWs {
  int* meta;        // Neff | Kc | order
  double* Kr64;     // [n][64][128]
  float* krimg;     // [n][16384]
  double* w64;      // [n][64]
  float *w32, *c32, *d32;
  unsigned* done;   // [n*batch]
  unsigned* flags;  // [S][ntiles]
  float* pub;       // [S][NL][ntiles*128][64]
  size_t bytes;
};
static FusedWs carve_fused(void* ws, int n, int64_t L, int batch, int S, int NL) {
  Carver c(ws);
  FusedWs w{};
  const int64_t ntiles = ceil_div(L, 128);
  w.meta = c.take<int>((size_t)3 * n);
  w.Kr64 = c.take<double>((size_t)n * 64 * 128);
  w.krimg = c.take<float>((size_t)n * 16384);
  w.w64 = c.take<double>((size_t)n * 64);
  w.w32 = c.take<float>((size_t)n * 64);
  w.c32 = c.take<float>((size_t)n * 64);
  w.d32 = c.take<float>((size_t)n);
  w.done = c.take<unsigned>((size_t)n * batch);
  w.flags = c.take<unsigned>((size_t)S * ntiles);
  w.pub = c.take<float>((size_t)S * NL * ntiles * 128 * 64);
  w.bytes = c.bytes();
  return w;
}
static int sm_count() {
  static const int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}
// sequence slots: enough for every sequence a CTA can be working on while others lag behind
static int fused_slots(int64_t nchunk, int64_t Q) {
  const int64_t s = 2 * ceil_div(148, nchunk) + 4;
  return (int)std::min<int64_t>(Q, s);
}
static size_t fused_ws_bytes(int n, int m, int64_t L, int batch, int n_max) {
  if (m != 64 || !fused_enabled()) return 0;
  const int NL = eff_order_b(n_max, L) - 6;
  if (NL < 1) return 0;
  const int64_t nchunk = ceil_div(ceil_div(L, 128), kFusedT);
  return carve_fused(nullptr, n, L, batch, fused_slots(nchunk, (int64_t)n * batch), NL).bytes;
}

size_t bank_ws_bytes(int n, int m, int64_t L, int batch, int n_max) {
  return std::max(carve_bank(nullptr, n, m, L, batch, stage_variant(m) == 't' ? pair_slots(n_max) : 0).bytes,
                  fused_ws_bytes(n, m, L, batch, n_max));
}

// Returns CASC_ERR_UNSUPPORTED when the fused path does not apply (caller falls back to the
// multi-kernel path), CASC_ERR_WORKSPACE when not even one sequence slot fits.
static int bank_fused(int n, int64_t L, int batch, const int* N_host, int N_max, const void* pack,
                      const double* Bbar, const double* C, const double* D, const void* u, void* y, void* ws,
                      size_t ws_bytes, cudaStream_t st) {
  constexpr int m = 64;
  if (!fused_enabled()) return CASC_ERR_UNSUPPORTED;
  const int64_t Q = (int64_t)n * batch;
  const int64_t ntiles = ceil_div(L, 128);
  if (Q >= (1 << 26) || ntiles >= (1 << 24)) return CASC_ERR_UNSUPPORTED;
  std::vector<int> meta((size_t)3 * n);
  int *Neff = meta.data(), *Kc = Neff + n, *order = Neff + 2 * n;
  int maxNe = 0;
  double flops = 0, bytes = 0;
  for (int s = 0; s < n; ++s) {
    Neff[s] = eff_order_b(N_host[s], L);
    if (Neff[s] < kHeadK) return CASC_ERR_UNSUPPORTED;
    Kc[s] = kHeadK;
    maxNe = std::max(maxNe, Neff[s]);
    flops += 2.0 * m * m * (N_host[s] + 1) * (double)L * batch;          // PAPER count, SURVEY 8d
    bytes += ((N_host[s] + 1) * 2.0 * m * 4.0 + 8.0) * (double)L * batch;  // unfused streaming bytes
  }
  std::iota(order, order + n, 0);
  std::stable_sort(order, order + n, [&](int a, int b) { return Neff[a] > Neff[b]; });
  const int NL = maxNe - 6;
  int T = kFusedT;
  if (const char* e = getenv("CASC_FUSED_T")) T = std::max(1, std::min(kFusedT, atoi(e)));
  const int64_t nchunk = ceil_div(ntiles, T);
  int S = fused_slots(nchunk, Q);
  if (const char* e = getenv("CASC_FUSED_SLOTS")) S = std::max(1, std::min(S, atoi(e)));   // tests: force reuse
  while (S > 1 && carve_fused(nullptr, n, L, batch, S, NL).bytes > ws_bytes) --S;
  FusedWs w = carve_fused(ws, n, L, batch, S, NL);
  if (w.bytes > ws_bytes) return CASC_ERR_WORKSPACE;
  PackLayout P = pack_layout(const_cast<void*>(pack), n, m, N_max, CASC_FP32);
  const int64_t mm = (int64_t)m * m;
  int rc;
  CASC_TRY(cudaMemcpyAsync(w.meta, meta.data(), meta.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  const int *dNeff = w.meta, *dKc = w.meta + n, *dorder = w.meta + 2 * n;
  {
    // derived: Krylov columns Kr[:, j] = Abar^j Bbar (j < 128) by doubling with the powers
    // (Kr_{2^i + j} = P_i Kr_j), their tf32 hi/lo smem image; w = C P_Ne; fp32 copies of C, D
    ProfScope ps(st, K_DERIVED, 0.0, 2.0 * n * (double)m * m * 128);
    if ((rc = launch_kr_init(Bbar, w.Kr64, n, m, st))) return rc;
    for (int i = 0; i < kHeadK; ++i) {
      DgemmArg a{};
      a.M = m; a.N = 1 << i; a.K = m;
      a.A = P.p64 + i * mm; a.lda = m; a.sA = (int64_t)(N_max + 1) * mm;
      a.B = w.Kr64; a.ldb = 128; a.sB = (int64_t)m * 128;
      a.C = w.Kr64 + (1 << i); a.ldc = 128; a.sC = (int64_t)m * 128;
      if ((rc = launch_dgemm(a, n, st))) return rc;
    }
    if ((rc = launch_kr_image(w.Kr64, dKc, w.krimg, n, st))) return rc;
    DgemmArg a{};                                // w = C P_Ne  (1 x m)
    a.M = 1; a.N = m; a.K = m;
    a.A = C; a.lda = m; a.sA = m;
    a.B = P.p64; a.ldb = m; a.sB = (int64_t)(N_max + 1) * mm; a.nB = mm; a.selB = dNeff;
    a.C = w.w64; a.ldc = m; a.sC = m;
    if ((rc = launch_dgemm(a, n, st))) return rc;
    if ((rc = launch_f64_to_f32(w.w64, w.w32, (int64_t)n * m, st))) return rc;
    if ((rc = launch_f64_to_f32(C, w.c32, (int64_t)n * m, st))) return rc;
    if (D) {
      if ((rc = launch_f64_to_f32(D, w.d32, n, st))) return rc;
    } else {
      CASC_TRY(cudaMemsetAsync(w.d32, 0, sizeof(float) * n, st));
    }
  }
  CASC_TRY(cudaMemsetAsync(w.done, 0, sizeof(unsigned) * (size_t)Q, st));
  CASC_TRY(cudaMemsetAsync(w.flags, 0, sizeof(unsigned) * (size_t)S * ntiles, st));
  BankFusedArg a{};
  a.u = static_cast<const float*>(u); a.y = static_cast<float*>(y); a.krimg = w.krimg;
  a.cvec = w.c32; a.wvec = w.w32; a.dvec = w.d32; a.order = dorder; a.Neff = dNeff;
  a.flags = w.flags; a.done = w.done; a.pub = w.pub;
  a.L = L; a.batch = batch; a.ntiles = (int)ntiles; a.T = T; a.nchunk = (int)nchunk; a.S = S; a.NL = NL;
  a.planes_per_ch = 2 * (N_max + 1); a.total_chunks = Q * nchunk; a.discard = discard_enabled() ? 1 : 0;
  const int grid = (int)std::min<int64_t>(a.total_chunks, sm_count());
  if (getenv("CASC_DEBUG"))
    fprintf(stderr, "casc: bank_fused n=%d L=%lld batch=%d ntiles=%lld nchunk=%lld S=%d NL=%d grid=%d ws=%zu\n", n,
            (long long)L, batch, (long long)ntiles, (long long)nchunk, S, NL, grid, w.bytes);
  static unsigned long long* dbg = nullptr;
  const bool want_dbg = getenv("CASC_FUSED_DBG") != nullptr;
  if (want_dbg) {
    if (!dbg) CASC_TRY(cudaMalloc(&dbg, 24 * sizeof(unsigned long long)));
    CASC_TRY(cudaMemsetAsync(dbg, 0, 24 * sizeof(unsigned long long), st));
    a.dbg = dbg;
  }
  {
    ProfScope ps(st, K_BANK_FUSED, bytes, flops);
    rc = launch_bank_fused(a, P.f32, (int)((int64_t)n * (N_max + 1) * 2), grid, st);
  }
  if (want_dbg && rc == CASC_OK) {          // diagnostics only: synchronises and prints
    unsigned long long h[24];
    CASC_TRY(cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, st));
    CASC_TRY(cudaStreamSynchronize(st));
    const double tot = (double)h[20] / grid;
    static const char* nm[5][4] = {{"prod.wfree/done", "prod.flag", "prod.aempty", "-"},
                                   {"mma.wfull", "mma.zfull", "mma.accempty", "mma.loready"},
                                   {"xf.done", "xf.zempty", "xf.afull", "xf.lofree"},
                                   {"epi.accfull", "epi.stg_empty", "epi.afull", "-"},
                                   {"st.stg_full", "st.read", "st.release", "-"}};
    fprintf(stderr, "casc fused dbg: grid %d, avg kernel cycles/CTA %.0f\n", grid, tot);
    for (int r = 0; r < 5; ++r)
      for (int i = 0; i < 4; ++i)
        if (h[r * 4 + i]) fprintf(stderr, "  %-16s %6.1f%%\n", nm[r][i], 100.0 * h[r * 4 + i] / grid / tot);
  }
  return rc;
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
  cudaStream_t cout = nullptr;      // copy-out stream
  cudaEvent_t u_ready = nullptr;    // input copy completion (the head waits for it)
  std::vector<cudaEvent_t>* events = nullptr;   // created here, destroyed by the caller
  // input arriving in chunks of channels [bounds[i], bounds[i+1]) (memory order), chunk i complete
  // at u_events[i]: the head runs per chunk as its input lands
  int n_chunks = 0; const int* bounds = nullptr; const cudaEvent_t* u_events = nullptr;
};
static int bank_wave(int n, int m, int64_t L, int batch, const int* N_host, int N_max, const PackLayout& Pw,
                     const double* Bbar, const double* C, const double* D, const float* u, float* y, void* ws,
                     size_t ws_bytes, cudaStream_t st, int* pinned_meta = nullptr, const BankStream* bs = nullptr);

// Bounded-memory bank: with a workspace smaller than the whole bank needs, the channels are
// processed in consecutive waves of as many channels as fit (each wave is an independent bank).
int engine_bank_tc(int n, int m, int64_t L, int batch, const int* N_host, int N_max, const void* pack,
                   const double* Bbar, const double* C, const double* D, const void* u, void* y, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  if (m == 64) {
    const int rc = bank_fused(n, L, batch, N_host, N_max, pack, Bbar, C, D, u, y, ws, ws_bytes, st);
    if (rc != CASC_ERR_UNSUPPORTED && rc != CASC_ERR_WORKSPACE) return rc;
  }
  int maxNe = 0;
  for (int s = 0; s < n; ++s) maxNe = std::max(maxNe, eff_order_b(N_host[s], L));
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

// End to end from host buffers with the transfers overlapped (casc_run_host, one wave): the input
// copy (copy-in stream) overlaps the parameter upload, the powers and the derived data, and each
// group of channels whose cascade is complete (the head for Ne <= 7, then every stage pass) gets
// its tail and its output copy (copy-out stream) while the remaining passes run. u_h / y_h should
// be pinned. CASC_ERR_WORKSPACE if the whole bank does not fit the workspace (caller falls back).
int engine_bank_pipelined(int n, int m, int64_t L, int batch, const int* N_host, int N_max, const void* pack,
                          const double* Bbar, const double* C, const double* D, float* u_dev, float* y_dev,
                          const void* u_h, const void* y_h, void* ws, size_t ws_bytes, cudaStream_t st) {
  int maxNe = 0;
  for (int s = 0; s < n; ++s) maxNe = std::max(maxNe, eff_order_b(N_host[s], L));
  const int qslots = stage_variant(m) == 't' ? pair_slots(maxNe) : 0;
  if (m != 64) return CASC_ERR_UNSUPPORTED;
  // channels per wave (bounded memory, as engine_bank_tc); every wave streams its own input chunks
  // and outputs, and wave w+1's input copy overlaps wave w's compute
  int nw = n;
  while (nw > 0 && carve_bank(nullptr, nw, m, L, batch, qslots).bytes > ws_bytes) {
    const size_t per = carve_bank(nullptr, 1, m, L, batch, qslots).bytes;
    nw = (int)std::min<size_t>((size_t)nw - 1, ws_bytes / std::max<size_t>(per, 1));
  }
  if (nw < 1) return CASC_ERR_WORKSPACE;
  static cudaStream_t out_streams[16] = {}, in_streams[16] = {};   // per device (created once)
  static int* pinned[16] = {};                     // per device pinned staging of the channel tables
  static size_t pinned_n[16] = {};
  int dev = 0;
  CASC_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 16) return CASC_ERR_UNSUPPORTED;
  if (!out_streams[dev]) CASC_TRY(cudaStreamCreateWithFlags(&out_streams[dev], cudaStreamNonBlocking));
  if (!in_streams[dev]) CASC_TRY(cudaStreamCreateWithFlags(&in_streams[dev], cudaStreamNonBlocking));
  if (pinned_n[dev] < (size_t)6 * n) {
    if (pinned[dev]) cudaFreeHost(pinned[dev]);
    pinned[dev] = nullptr;
    pinned_n[dev] = 0;
    CASC_TRY(cudaHostAlloc(&pinned[dev], sizeof(int) * 6 * (size_t)n, cudaHostAllocDefault));
    pinned_n[dev] = (size_t)6 * n;
  }
  std::vector<cudaEvent_t> events;
  auto new_event = [&](cudaEvent_t* e) -> int {
    CASC_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    events.push_back(*e);
    return CASC_OK;
  };
  cudaEvent_t ev_start;
  int rc = new_event(&ev_start);
  if (rc) return rc;
  // u may be overwritten only after earlier work on st (starting the copy before the parameter
  // copies and powers measured slower on E2: 5.48 vs 4.26 ms e2e)
  CASC_TRY(cudaEventRecord(ev_start, st));
  CASC_TRY(cudaStreamWaitEvent(in_streams[dev], ev_start, 0));
  const bool timing = getenv("CASC_TIMING") && g_timing_t0;  // diagnostics: copy-in timeline
  cudaEvent_t t_start = nullptr, t_in0 = nullptr;
  if (timing) {
    cudaEventCreate(&t_start); cudaEventCreate(&t_in0);
    cudaEventRecord(t_start, in_streams[dev]);
  }
  const size_t row = (size_t)batch * L * sizeof(float);
  const int waves = (n + nw - 1) / nw;
  std::vector<std::vector<int>> bounds(waves);
  std::vector<std::vector<cudaEvent_t>> u_ev(waves);
  // input copies of wave w, submitted just before the wave's own work: a small host->device copy
  // the wave enqueues (its channel table) queues behind every copy submitted before it on the
  // copy engine, so submitting all waves' inputs up front delayed wave 0 by the whole input (E5:
  // 140 ms); wave w+1's copy still runs during wave w's compute
  for (int w = 0; w < waves; ++w) {                // chunk bounds and completion events of every wave
    static const int chunks = [] {                  // input chunks per wave (CASC_E2E_CHUNKS)
      const char* e = getenv("CASC_E2E_CHUNKS");
      return e ? std::max(1, atoi(e)) : 1;   // measured: 1 chunk 4.48 ms e2e on E2, 8 chunks 4.80
    }();
    const int c0 = w * nw, cn = std::min(nw, n - c0), nc = std::min(cn, chunks);
    bounds[w].resize(nc + 1);
    u_ev[w].resize(nc);
    for (int i = 0; i <= nc; ++i) bounds[w][i] = (int)((int64_t)cn * i / nc);
    for (int i = 0; i < nc; ++i)
      if ((rc = new_event(&u_ev[w][i]))) return rc;
  }
  auto submit_inputs = [&](int w) -> int {
    const int c0 = w * nw, nc = (int)u_ev[w].size();
    for (int i = 0; i < nc; ++i) {
      const size_t off = (size_t)(c0 + bounds[w][i]) * row;
      CASC_TRY(cudaMemcpyAsync((char*)u_dev + off, (const char*)u_h + off, (size_t)(bounds[w][i + 1] - bounds[w][i]) * row,
                               cudaMemcpyHostToDevice, in_streams[dev]));
      CASC_TRY(cudaEventRecord(u_ev[w][i], in_streams[dev]));
      if (timing && w == 0 && i == nc - 1) cudaEventRecord(t_in0, in_streams[dev]);
    }
    return CASC_OK;
  };
  PackLayout P = pack_layout(const_cast<void*>(pack), n, m, N_max, CASC_FP32);
  const int64_t slot_mm = (int64_t)(N_max + 1) * m * m;
  for (int w = 0; w < waves && rc == CASC_OK; ++w) {
    if ((rc = submit_inputs(w))) break;
    const int c0 = w * nw, cn = std::min(nw, n - c0);
    BankStream bs;
    bs.y_host = (char*)const_cast<void*>(y_h) + (size_t)c0 * row;
    bs.cout = out_streams[dev];
    bs.events = &events;
    bs.n_chunks = (int)u_ev[w].size();
    bs.bounds = bounds[w].data();
    bs.u_events = u_ev[w].data();
    PackLayout Pw = P;
    Pw.p64 += c0 * slot_mm;
    Pw.f32 += c0 * slot_mm * 2;
    const int64_t sig = (int64_t)c0 * batch * L;
    rc = bank_wave(cn, m, L, batch, N_host + c0, N_max, Pw, Bbar + (int64_t)c0 * m, C + (int64_t)c0 * m,
                   D ? D + c0 : nullptr, u_dev + sig, y_dev + sig, ws, ws_bytes, st, pinned[dev] + 6 * (size_t)c0, &bs);
  }
  if (getenv("CASC_TIMING") && g_timing_t0) {       // diagnostics: when each stream finishes
    cudaEvent_t a, b, c;
    cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&c);
    cudaEventRecord(a, in_streams[dev]); cudaEventRecord(b, st); cudaEventRecord(c, out_streams[dev]);
    cudaDeviceSynchronize();
    float ta, tb, tc;
    cudaEventElapsedTime(&ta, g_timing_t0, a); cudaEventElapsedTime(&tb, g_timing_t0, b); cudaEventElapsedTime(&tc, g_timing_t0, c);
    fprintf(stderr, "casc timing: input copies done %.3f, compute done %.3f, output copies done %.3f ms\n", ta, tb, tc);
    if (t_start && t_in0) {
      float t0s, t0i;
      cudaEventElapsedTime(&t0s, g_timing_t0, t_start); cudaEventElapsedTime(&t0i, g_timing_t0, t_in0);
      fprintf(stderr, "casc timing: copy-in starts %.3f, wave 0 input landed %.3f ms\n", t0s, t0i);
      cudaEventDestroy(t_start); cudaEventDestroy(t_in0);
    }
    cudaEventDestroy(a); cudaEventDestroy(b); cudaEventDestroy(c);
  }
  cudaError_t e1 = cudaStreamSynchronize(out_streams[dev]), e2 = cudaStreamSynchronize(st);
  cudaError_t e3 = cudaStreamSynchronize(in_streams[dev]);
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
  // v (R24); taken with the m = 64 TMA stage GEMM and warp-specialized head
  static const bool ab_off = [] {
    const char* e = getenv("CASC_BANK_AB");
    return e && e[0] == '0';
  }();
  const bool use_ab = m == 64 && (variant == 's' || variant == 't') && !ab_off && !(getenv("CASC_BANK_HEAD") && getenv("CASC_BANK_HEAD")[0] == 'o');
  std::vector<int> meta_v(pinned_meta ? 0 : (size_t)6 * n);
  int* meta = pinned_meta ? pinned_meta : meta_v.data();
  int *Neff = meta, *Kc = Neff + n, *par = Neff + 2 * n, *order = Neff + 3 * n, *iota = Neff + 4 * n,
      *hend = Neff + 5 * n;
  int maxNe = 0;
  for (int s = 0; s < n; ++s) {
    Neff[s] = eff_order_b(N_host[s], L);
    Kc[s] = std::min(kHeadK, Neff[s]);
    const int nstream = Neff[s] - Kc[s];            // streaming stages of this channel
    par[s] = (variant == 't' ? (nstream + 1) / 2 : nstream) % 2;   // passes -> final buffer
    maxNe = std::max(maxNe, Neff[s]);
  }
  const int qslots = variant == 't' ? pair_slots(maxNe) : 0;
  BankWs w = carve_bank(ws, n, m, L, batch, qslots);
  if (ws_bytes < w.bytes) {
    if (getenv("CASC_DEBUG")) fprintf(stderr, "casc: bank wave ws=%zu need=%zu n=%d\n", ws_bytes, w.bytes, n);
    return CASC_ERR_WORKSPACE;
  }
  const PackLayout& P = Pw;
  const int64_t mm = (int64_t)m * m;
  int rc;
  std::iota(order, order + n, 0);
  std::stable_sort(order, order + n, [&](int a, int b) { return Neff[a] > Neff[b]; });
  std::iota(iota, iota + n, 0);
  // R24-R26 (common.cuh OutParts): y is formed from parts written by the kernel producing
  // v^(Ne-d); with fold, d = 1 for an odd number of streaming stages (no single-stage pass) and
  // d = 2 for an even number >= 2 (the last stage-pair pass is skipped). Planned only where every
  // pass producing d > 0 parts runs on the history-resident kernel (or is the head).
  // CASC_BANK_FOLD = 0 | 1 (R25, default) | 2 (R25 + R26: measured slower, E2 3.90 vs 3.75 ms and
  // E5 807 vs 768 ms, the eight-part epilogues cost more than the skipped pair passes save)
  static const int fold_mode = [] {
    const char* e = getenv("CASC_BANK_FOLD");
    return e ? atoi(e) : 1;
  }();
  int fold = (use_ab && variant == 't') ? fold_mode : 0;
  for (int c = 0; fold && c < n; ++c) {
    const int d = fold_depth(Neff[c], Kc[c], fold), lp = Neff[c] - d;
    if (d > 0 && lp > Kc[c] && !bank_hist_ok(L, (int64_t)1 << (lp - 2), 3, 0)) fold = 0;
  }
  std::vector<int> Lp(n);                          // the state level each channel's parts come from
  for (int c = 0; c < n; ++c) Lp[c] = Neff[c] - fold_depth(Neff[c], Kc[c], fold);
  auto ends_at_head = [&](int c) { return Lp[c] == Kc[c]; };
  const bool chunked = bs && bs->n_chunks > 1;
  std::vector<int> hend_off(chunked ? bs->n_chunks + 1 : 1, 0);
  if (chunked) {                                   // head-ending channels (Ne == Kc), grouped by chunk
    int o = 0;
    for (int ci = 0; ci < bs->n_chunks; ++ci) {
      hend_off[ci] = o;
      for (int c = bs->bounds[ci]; c < bs->bounds[ci + 1]; ++c)
        if (ends_at_head(c)) hend[o++] = c;
    }
    hend_off[bs->n_chunks] = o;
  }
  CASC_TRY(cudaMemcpyAsync(w.meta, meta, (size_t)6 * n * sizeof(int), cudaMemcpyHostToDevice, st));
  const int *dNeff = w.meta, *dKc = w.meta + n, *dpar = w.meta + 2 * n, *dorder = w.meta + 3 * n,
            *diota = w.meta + 4 * n, *dhend = w.meta + 5 * n;
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
    static cudaStream_t q_streams[16] = {};
    int qdev = 0;
    CASC_TRY(cudaGetDevice(&qdev));
    if (qdev < 0 || qdev >= 16) return CASC_ERR_UNSUPPORTED;
    if (!q_streams[qdev]) CASC_TRY(cudaStreamCreateWithFlags(&q_streams[qdev], cudaStreamNonBlocking));
    qs = q_streams[qdev];
    CASC_TRY(cudaEventCreateWithFlags(&q_start, cudaEventDisableTiming));
    CASC_TRY(cudaEventCreateWithFlags(&q_done, cudaEventDisableTiming));
    CASC_TRY(cudaEventRecord(q_start, st));
    CASC_TRY(cudaStreamWaitEvent(qs, q_start, 0));
    ProfScope ps(st, K_DERIVED, 0.0, 2.0 * n * (double)m * m * 128);
    if ((rc = launch_bank_derived(P.p64, N_max + 1, Bbar, C, D, dNeff, dKc, w.Kr64, w.krT, w.w64, w.w32, w.c32,
                                  w.d32, use_ab ? w.pvec : nullptr, fold, n, m, st)))
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
  auto emit_ids = [&](const int* dlist, const int* hlist, int cnt) -> int {
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
    for (int i = 0; i < cnt;) {                   // merge runs of consecutive channel ids
      int j = i + 1;
      while (j < cnt && hlist[j] == hlist[j - 1] + 1) ++j;
      CASC_TRY(cudaMemcpyAsync((char*)bs->y_host + (size_t)hlist[i] * row, (const char*)y + (size_t)hlist[i] * row,
                               (size_t)(j - i) * row, cudaMemcpyDeviceToHost, bs->cout));
      i = j;
    }
    return CASC_OK;
  };
  auto emit = [&](int a, int b) -> int { return emit_ids(dorder + a, order + a, b - a); };
  // ---- head: stages 0..Kc-1 (+ Bbar u), all channels (per input chunk when the input is streamed)
  if (bs && bs->u_ready) CASC_TRY(cudaStreamWaitEvent(st, bs->u_ready, 0));
  for (int ci = 0; ci < (chunked ? bs->n_chunks : 1); ++ci) {
    if (chunked) CASC_TRY(cudaStreamWaitEvent(st, bs->u_events[ci], 0));
    const int hc0 = chunked ? bs->bounds[ci] : 0, hcn = chunked ? bs->bounds[ci + 1] - hc0 : n;
    BankHeadArg a{};
    a.u = static_cast<const float*>(u); a.krT = w.krT; a.V = static_cast<float*>(w.Va);
    a.sys_list = chunked ? diota + hc0 : dorder; a.n_list = hcn; a.L = L; a.batch = batch;
    if (use_ab) a.op = op;
    a.tiles_per_cta = pick_group(ntiles, (int64_t)n * batch, 16);
    ProfScope ps(st, K_BANK_HEAD, (double)n * batch * L * (1 + m) * 4.0,
                 (double)n * batch * L * 2.0 * m * 128);
    // warp-specialized TMA-store head for m = 64 (CASC_BANK_HEAD=old selects the previous kernel).
    // A TMEM-operand (TS) variant was measured slower (1.67 vs 1.30 ms on E2, same box): its four
    // builder warps write 128 KB of hi/lo per tile to TMEM.
    // CASC_BANK_HEAD = ws (default: one CTA per tile) | pair (CTA pairs, M = 256: measured the same
    // 1.16 ms on E2 -- the head is bound by the tensor pipe, 69% active, not by operand reads) | old
    static const char head_kind = [] {
      const char* e = getenv("CASC_BANK_HEAD");
      return e ? e[0] : 'w';
    }();
    const bool old_head = head_kind == 'o';
    static const int head_group = [] {
      const char* e = getenv("CASC_HEAD_GROUP");
      return e ? atoi(e) : 64;
    }();
    if (m == 64 && !old_head) a.tiles_per_cta = pick_group(ntiles, (int64_t)hcn * batch, head_group);
    if (m == 64 && !old_head)
      rc = head_kind == 'p' ? launch_bank_head_pair(m, a, (int64_t)n * batch, st)
                            : launch_bank_head_ws(m, a, (int64_t)n * batch, st);
    else
      rc = launch_bank_head(m, a, st);
    if (rc) return rc;
    if (chunked && (rc = emit_ids(dhend + hend_off[ci], hend + hend_off[ci], hend_off[ci + 1] - hend_off[ci])))
      return rc;
  }
  // cascades whose output parts come from the head (Ne <= 7; with fold also Ne = 8, 9)
  if (!chunked && (rc = emit(count_lp_ge(kHeadK + 1), n))) return rc;
  auto tmark = [&](const char* what) {              // CASC_TIMING diagnostics
    if (!getenv("CASC_TIMING") || !g_timing_t0) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    cudaEventSynchronize(e);
    float t;
    cudaEventElapsedTime(&t, g_timing_t0, e);
    fprintf(stderr, "casc timing: %s %.3f ms\n", what, t);
    cudaEventDestroy(e);
  };
  tmark("head done");
  if (q_done) CASC_TRY(cudaStreamWaitEvent(st, q_done, 0));   // the pair weights
  // ---- streaming stages k >= kHeadK over the channels with Neff > k (prefixes of `order`)
  int pass = 0;
  for (int k = kHeadK; k < maxNe; k += (variant == 't' ? 2 : 1), ++pass) {
    const float* Vs = static_cast<const float*>(pass % 2 == 0 ? w.Va : w.Vb);
    float* Vd = static_cast<float*>(pass % 2 == 0 ? w.Vb : w.Va);
    if (variant == 's') {                           // TMA GEMM, one stage per pass
      const int cnt = count_ge(k + 1);
      MimoGemm g{};
      g.src[0].A = Vs; g.src[0].W = P.f32; g.src[0].K = m; g.src[0].shift = (int64_t)1 << k;
      g.src[0].w_plane_off = 2 * k; g.src[0].w_planes = (int64_t)n * (N_max + 1) * 2;
      g.src[0].w_plane_stride = 2 * (N_max + 1);
      g.n_src = 1; g.R = Vs; g.out = Vd; g.n_out = m; g.L = L; g.batch = batch;
      g.sys_list = dorder; g.n_list = cnt; g.n_sys_total = n;
      g.t_first = pass == 0 ? 0 : (int)(((int64_t)1 << (k - 1)) / 128);
      g.w_resident = resident_weights();
      if (use_ab) {                                 // channels whose last streaming stage this is
        g.ab_neff = dNeff; g.ab_level = k + 1; g.ab_c = w.c32; g.ab_w = w.w32; g.ab = w.parts; g.ab_plane = plane;
        // their (C v, C P_Ne v) parts are needed on every row: no skipped leading tiles
        if (count_ge(k + 1) > count_ge(k + 2)) g.t_first = 0;
      }
      {
        ProfScope ps(st, K_BANK_STAGE, 2.0 * cnt * batch * L * m * 4.0, 2.0 * cnt * batch * L * (double)mm);
        if ((rc = launch_mimo_gemm(g, true, st))) return rc;
      }
      if ((rc = emit(count_ge(k + 2), count_ge(k + 1)))) return rc;   // channels with Ne == k + 1
      continue;
    }
    if (variant != 't') {
      const int cnt = count_ge(k + 1);
      BankStageArg a{};
      a.Vs = Vs; a.Vd = Vd; a.P = P.f32; a.k = k; a.slots = N_max + 1;
      a.copy_from = (k == kHeadK) ? 0 : ((int64_t)1 << (k - 1));
      a.sys_list = dorder; a.n_list = cnt; a.L = L; a.batch = batch;
      a.tiles_per_cta = pick_group(ntiles, (int64_t)cnt * batch, 8);
      ProfScope ps(st, K_BANK_STAGE, 2.0 * cnt * batch * L * m * 4.0, 2.0 * cnt * batch * L * (double)mm);
      rc = variant == 'w' ? launch_bank_stage_ws(m, a, st) : launch_bank_stage_rp(m, a, st);
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
      g.sys_list = dorder; g.n_list = cnt2; g.n_sys_total = n; g.t_first = t_first; g.w_resident = pair_wres();
      if (use_ab) {                                 // channels whose parts come from this pass (Lp == k + 2)
        g.ab_neff = dNeff; g.ab_level = k + 2; g.ab_c = w.c32; g.ab_w = w.w32; g.ab = w.parts; g.ab_plane = plane;
        g.parts = op; g.parts.level = k + 2;
        for (int c = 0; c < n; ++c) g.parts_deep |= (Lp[c] == k + 2 && Lp[c] != Neff[c]);
        if (count_lp_ge(k + 2) > count_lp_ge(k + 3)) g.t_first = 0;   // their parts need every row
      }
      // bytes of the schedule run (SURVEY 8d B_fused): one read + one write of the state for the two
      // stages this pass applies; flops of both stages (bench.py derives the unfused B_ns from them)
      ProfScope ps(st, K_BANK_STAGE, 2.0 * cnt2 * batch * L * m * 4.0, 4.0 * cnt2 * batch * L * (double)mm);
      rc = launch_bank_hist(g, st);
      if (rc == CASC_ERR_UNSUPPORTED) rc = launch_mimo_gemm(g, true, st);
      if (rc) return rc;
    }
    if (cnt1 > 0) {                                // single stage k for Ne == k + 1 (none with fold)
      MimoGemm g{};
      g.src[0].A = Vs; g.src[0].W = P.f32; g.src[0].K = m; g.src[0].shift = (int64_t)1 << k;
      g.src[0].w_plane_off = 2 * k; g.src[0].w_planes = planes; g.src[0].w_plane_stride = 2 * (N_max + 1);
      g.n_src = 1; g.R = Vs; g.out = Vd; g.n_out = m; g.L = L; g.batch = batch;
      g.sys_list = dorder + cnt2; g.n_list = cnt1; g.n_sys_total = n; g.t_first = t_first; g.w_resident = resident_weights();
      if (use_ab) {                                 // every channel here ends with stage k
        g.ab_neff = dNeff; g.ab_level = k + 1; g.ab_c = w.c32; g.ab_w = w.w32; g.ab = w.parts; g.ab_plane = plane;
        g.parts = op; g.parts.level = k + 1;
        g.t_first = 0;
      }
      ProfScope ps(st, K_BANK_STAGE, 2.0 * cnt1 * batch * L * m * 4.0, 2.0 * cnt1 * batch * L * (double)mm);
      rc = launch_bank_hist(g, st);
      if (rc == CASC_ERR_UNSUPPORTED) rc = launch_mimo_gemm(g, true, st);
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
