// Host sequencing of the MIMO tensor-core path (one system; m, p, q multiples of 64).
// Same step schedule as the generic engine (cascade_api.cu), each step one launch of the
// shifted multi-source tcgen05 GEMM (mimo_tc.cu), in bf16 or 3xTF32 (fp32 mode):
//   Ne == 0 : y = (C Bbar + D) u_l + (C Abar Bbar) u_{l-1}
//   first   : v^(1) = Bbar u_l + Abar Bbar u_{l-1}                       -> Va
//   stage k : v^(k+1) = v^(k) + P_k v^(k)_{l-2^k},  k = 1 .. Ne-1          Va <-> Vb
//   last    : y = C v + (C P_Ne) v_{l-2^Ne} + D u
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"
#include "engine.cuh"
#include "mimo_tc.cuh"
#include "profile.cuh"

namespace casc {

MimoWs carve_mimo(void* ws, int m, int p, int q, int64_t L, int batch, int mode) {
  Carver c(ws);
  MimoWs w{};
  const size_t wes = mode == CASC_FP32 ? 8 : 2;      // tf32 hi+lo pair, or bf16
  const size_t ses = mode == CASC_FP32 ? 4 : 2;      // signal element size
  w.AB64 = c.take<double>((size_t)m * p);
  w.CP64 = c.take<double>((size_t)q * m);
  w.CBD64 = c.take<double>((size_t)q * p);
  w.CAB64 = c.take<double>((size_t)q * p);
  w.A2B64 = c.take<double>((size_t)m * p);
  w.A3B64 = c.take<double>((size_t)m * p);
  w.CP1_64 = c.take<double>((size_t)q * m);
  w.CP3_64 = c.take<double>((size_t)q * m);
  w.Bb = c.take<char>((size_t)m * p * wes);
  w.AB = c.take<char>((size_t)m * p * wes);
  w.C = c.take<char>((size_t)q * m * wes);
  w.CP = c.take<char>((size_t)q * m * wes);
  w.D = c.take<char>((size_t)q * p * wes);
  w.CBD = c.take<char>((size_t)q * p * wes);
  w.CAB = c.take<char>((size_t)q * p * wes);
  w.A2B = c.take<char>((size_t)m * p * wes);
  w.A3B = c.take<char>((size_t)m * p * wes);
  w.CP1 = c.take<char>((size_t)q * m * wes);
  w.CP3 = c.take<char>((size_t)q * m * wes);
  const size_t vbytes = (size_t)batch * (size_t)L * m * ses;
  w.Va = c.take<char>(vbytes);
  w.Vb = c.take<char>(vbytes);
  w.bytes = c.bytes();
  return w;
}

bool mimo_tc_path(int n, int m, int p, int q, int mode) {
  static const bool force_simt = [] {
    const char* e = getenv("CASC_FORCE_SIMT");
    return e && e[0] == '1';
  }();
  return !force_simt && n == 1 && mimo_tc_supported(m, p, q);
}

size_t mimo_ws_bytes(int m, int p, int q, int64_t L, int batch, int mode) {
  return carve_mimo(nullptr, m, p, q, L, batch, mode).bytes;
}


int engine_mimo_tc(int m, int p, int q, int64_t L, int batch, int N, int N_max, int mode, const void* pack,
                   const double* Bbar, const double* C, const double* D, const void* u, void* y, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  MimoWs w = carve_mimo(ws, m, p, q, L, batch, mode);
  if (ws_bytes < w.bytes) return CASC_ERR_WORKSPACE;
  PackLayout P = pack_layout(const_cast<void*>(pack), 1, m, N_max, mode);
  const int Ne = eff_order(N, L);
  int rc;
  if ((rc = mimo_derive(m, p, q, Ne, P, Bbar, C, D, w, mode == CASC_FP32, st))) return rc;
  return mimo_run(m, p, q, L, batch, Ne, N_max, mode, pack, D != nullptr, u, y, 0, ws, ws_bytes, st);
}

// The cascade steps of one MIMO system on `batch` sequences of L rows, derived weights already in
// ws (mimo_derive). out_skip > 0 (one sequence only): a window whose first out_skip rows are input
// history -- y is written for rows [out_skip, L) only, to y (which points at the first kept row);
// exact when out_skip >= 2^(Ne+1) - 1 or the window starts at the sequence start (PAPER.md:137-141,
// pin T14).
int mimo_run(int m, int p, int q, int64_t L, int batch, int Ne, int N_max, int mode, const void* pack, bool has_D,
             const void* u, void* y, int64_t out_skip, void* ws, size_t ws_bytes, cudaStream_t st) {
  MimoWs w = carve_mimo(ws, m, p, q, L, batch, mode);
  if (ws_bytes < w.bytes) return CASC_ERR_WORKSPACE;
  if (out_skip < 0 || out_skip >= L || (out_skip > 0 && (batch != 1 || Ne == 0))) return CASC_ERR_ARG;
  const bool tf32 = mode == CASC_FP32;
  PackLayout P = pack_layout(const_cast<void*>(pack), 1, m, N_max, mode);
  const int64_t mm = (int64_t)m * m;
  const double es = tf32 ? 4.0 : 2.0;
  int rc;
  const double rows = (double)batch * L, yrows = (double)batch * (L - out_skip);
  const double xf = tf32 ? 3.0 : 1.0;            // executed products per source: 3xTF32 or one bf16
  const int pipe = tf32 ? PIPE_TF32 : PIPE_BF16;
  if (Ne == 0) {
    MimoGemm g{};
    g.src[0] = {u, w.CBD, p, 0};
    g.src[1] = {u, w.CAB, p, 1};
    g.n_src = 2; g.out = y; g.n_out = q; g.L = L; g.batch = batch;
    ProfScope ps(st, K_MIMO_LAST, rows * (p + q) * es, rows * 4.0 * q * p);
    ps.exec(rows * (p + q) * es, rows * 4.0 * q * p * xf, pipe);
    return launch_mimo_gemm(g, tf32, st);
  }
  // a2 + a3: the Krylov head (R28) -- v^(2)_l = sum_{j<4} (Abar^j Bbar) u_{l-j}, the expanded product
  // of Bbar u and the factors k = 0, 1 of Eq. 5, one 4-source GEMM with K = 4p instead
  // of the first step (K = 2p) and stage 1 (K = m); with Ne = 1 the fused first step alone
  const int k0 = Ne >= 2 ? 2 : 1;                // first streaming stage
  {
    MimoGemm g{};
    g.src[0] = {u, w.Bb, p, 0};
    g.src[1] = {u, w.AB, p, 1};
    g.n_src = 2;
    if (k0 == 2) {
      g.src[2] = {u, w.A2B, p, 2};
      g.src[3] = {u, w.A3B, p, 3};
      g.n_src = 4;
    }
    g.out = k0 == 2 ? w.Vb : w.Va; g.n_out = m; g.L = L; g.batch = batch;
    ProfScope ps(st, K_MIMO_FIRST, rows * (p + m) * es, rows * 2.0 * g.n_src * m * p);
    ps.exec(rows * (p + m) * es, rows * 2.0 * g.n_src * m * p * xf, pipe);
    if ((rc = launch_mimo_gemm(g, tf32, st))) return rc;
  }
  const int kl = mimo_fold(Ne) ? Ne - 1 : Ne;     // the state level the output step reads (R31)
  for (int k = k0; k <= kl - 1; ++k) {
    void* Vs = (k - 1) % 2 == 0 ? w.Va : w.Vb;
    void* Vd = (k % 2 == 0) ? w.Va : w.Vb;
    // stage weight P_k: bf16 [m][m] or the tf32 pair [2][m][m] of the pack
    const void* Wk = tf32 ? static_cast<const void*>(P.f32 + k * 2 * mm) : static_cast<const void*>(P.b16 + k * mm);
    MimoGemm g{};
    g.src[0] = {Vs, Wk, m, (int64_t)1 << k};
    g.n_src = 1; g.R = Vs; g.out = Vd; g.n_out = m; g.L = L; g.batch = batch;
    ProfScope ps(st, K_MIMO_STAGE, rows * m * es * 2.0, rows * 2.0 * (double)mm);
    ps.exec(rows * m * es * 2.0 + (double)mm * (tf32 ? 8.0 : 2.0), rows * 2.0 * (double)mm * xf, pipe);
    if ((rc = launch_mimo_gemm(g, tf32, st))) return rc;
  }
  {
    void* V = (kl - 1) % 2 == 0 ? w.Va : w.Vb;     // holds v^(kl)
    MimoGemm g{};
    mimo_output_gemm(g, w, Ne, m, p, q, V, out_skip, u, out_skip, has_D, 1);
    g.out = y; g.n_out = q; g.L = L - out_skip; g.batch = batch;
    const double k_in = (double)(g.n_src - (has_D ? 1 : 0)) * m + (has_D ? p : 0);
    ProfScope ps(st, K_MIMO_LAST, yrows * (m + p + q) * es, yrows * 2.0 * q * k_in);
    ps.exec(yrows * (m + p + q) * es, yrows * 2.0 * q * k_in * xf, pipe);
    if ((rc = launch_mimo_gemm(g, tf32, st))) return rc;
  }
  return CASC_OK;
}

void mimo_output_gemm(MimoGemm& g, const MimoWs& w, int Ne, int m, int p, int q, const void* V, int64_t v_row0,
                      const void* u, int64_t u_row0, bool has_D, int64_t unit) {
  (void)q;
  if (mimo_fold(Ne)) {
    const int64_t h = ((int64_t)1 << (Ne - 1)) * unit;
    g.src[0] = {V, w.C, m, 0};
    g.src[1] = {V, w.CP1, m, h};
    g.src[2] = {V, w.CP, m, 2 * h};
    g.src[3] = {V, w.CP3, m, 3 * h};
    g.n_src = 4;
  } else {
    g.src[0] = {V, w.C, m, 0};
    g.src[1] = {V, w.CP, m, ((int64_t)1 << Ne) * unit};
    g.n_src = 2;
  }
  for (int i = 0; i < g.n_src; ++i) g.src[i].row0 = v_row0;
  if (has_D) {
    g.src[g.n_src] = {u, w.D, p, 0};
    g.src[g.n_src].row0 = u_row0;
    ++g.n_src;
  }
}

// Derived weights of the fused first / last steps (R21, R28, R31), in float64, then rounded
// once to the GEMM operand format -- all in ONE cooperative launch (launch_derived_coop, dgemm.cu):
//   phase 1: Abar Bbar, Abar^2 Bbar = P_1 Bbar, C P_Ne, C P_{Ne-1}, C Bbar + D
//   phase 2: Abar^3 Bbar = P_1 (Abar Bbar), (C P_Ne) P_{Ne-1}, C (Abar Bbar)
//   phase 3: every weight to tf32 hi/lo planes (fp32 mode) or bf16
int mimo_derive(int m, int p, int q, int Ne, const PackLayout& P, const double* Bbar, const double* C,
                const double* D, const MimoWs& w, bool tf32, cudaStream_t st) {
  const int64_t mm = (int64_t)m * m;
  DerivedPlan pl{};
  auto job = [&](int ph, const double* A, int lda, const double* B, int ldb, double* Cm, int ldc, int M, int N,
                 const double* Cadd) {
    DJob& j = pl.jobs[pl.n_jobs++];
    j = DJob{A, B, Cm, Cadd, lda, ldb, ldc, M, N, m, ph};
  };
  auto cvt = [&](const double* src, void* dst, int64_t n) {
    DConv& c = pl.convs[pl.n_convs++];
    c = DConv{src, dst, n};
  };
  job(0, P.p64, m, Bbar, p, w.AB64, p, m, p, nullptr);                          // Abar Bbar
  job(0, C, m, P.p64 + Ne * mm, m, w.CP64, m, q, m, nullptr);                  // C P_Ne
  job(0, C, m, Bbar, p, w.CBD64, p, q, p, D);                                   // C Bbar + D
  job(1, C, m, w.AB64, p, w.CAB64, p, q, p, nullptr);                           // C Abar Bbar
  cvt(Bbar, w.Bb, (int64_t)m * p);
  cvt(w.AB64, w.AB, (int64_t)m * p);
  cvt(C, w.C, (int64_t)q * m);
  cvt(w.CP64, w.CP, (int64_t)q * m);
  cvt(w.CBD64, w.CBD, (int64_t)q * p);
  cvt(w.CAB64, w.CAB, (int64_t)q * p);
  if (D) cvt(D, w.D, (int64_t)q * p);
  if (Ne >= 2) {                                                                // Krylov head (R28)
    job(0, P.p64 + mm, m, Bbar, p, w.A2B64, p, m, p, nullptr);                 // P_1 Bbar
    job(1, P.p64 + mm, m, w.AB64, p, w.A3B64, p, m, p, nullptr);               // P_1 (Abar Bbar)
    cvt(w.A2B64, w.A2B, (int64_t)m * p);
    cvt(w.A3B64, w.A3B, (int64_t)m * p);
  }
  if (mimo_fold(Ne)) {                                                          // output fold (R31)
    job(0, C, m, P.p64 + (Ne - 1) * mm, m, w.CP1_64, m, q, m, nullptr);        // C P_{Ne-1}
    job(1, w.CP64, m, P.p64 + (Ne - 1) * mm, m, w.CP3_64, m, q, m, nullptr);   // (C P_Ne) P_{Ne-1}
    cvt(w.CP1_64, w.CP1, (int64_t)q * m);
    cvt(w.CP3_64, w.CP3, (int64_t)q * m);
  }
  pl.tf32 = tf32 ? 1 : 0;
  double fl = 0.0;
  for (int i = 0; i < pl.n_jobs; ++i) fl += 2.0 * pl.jobs[i].M * pl.jobs[i].N * pl.jobs[i].K;
  ProfScope ps(st, K_DERIVED, 0.0, fl);
  ps.exec(0.0, fl, PIPE_FP64);
  return launch_derived_coop(pl, st);
}

}  // namespace casc
