// Host sequencing of the tensor-core bank path (SISO channels, fp32 mode, m in {16, 32, 64}).
//   derived : Krylov columns Abar^j Bbar (j < 2^Kc) by doubling with the powers
//             [Kr_{2^i + j} = P_i Kr_j], tf32 hi/lo image; w = C P_Ne; fp32 copies of C, D
//   head    : v^(Kc) (stages 0..Kc-1 with Bbar u)          -> Va
//   stage k : k = Kc .. Ne-1 (only channels with Ne > k)   Va <-> Vb
//   tail    : stage Ne + y = C v + D u                      -> y
#include <algorithm>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "bank_tc.cuh"
#include "profile.cuh"
#include "engine.cuh"
#include "mimo_tc.cuh"

namespace casc {

static constexpr int kHeadK = 7;      // Krylov head covers stages 0..6 (128 lags)

struct BankWs {
  int* meta;      // Neff | Kc | parity | order   (4 n ints)
  double* Kr64;   // [n][m][128]
  float* krT;     // [n][2][m][128]
  double* w64;    // [n][m]
  float *w32, *c32, *d32;
  void *Va, *Vb;
  size_t bytes;
};

static BankWs carve_bank(void* ws, int n, int m, int64_t L, int batch) {
  Carver c(ws);
  BankWs w{};
  w.meta = c.take<int>((size_t)4 * n);
  w.Kr64 = c.take<double>((size_t)n * m * 128);
  w.krT = c.take<float>((size_t)n * 2 * m * 128);
  w.w64 = c.take<double>((size_t)n * m);
  w.w32 = c.take<float>((size_t)n * m);
  w.c32 = c.take<float>((size_t)n * m);
  w.d32 = c.take<float>((size_t)n);
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

size_t bank_ws_bytes(int n, int m, int64_t L, int batch) { return carve_bank(nullptr, n, m, L, batch).bytes; }

static int eff_order_b(int N, int64_t L) {
  if (L <= 2) return 0;
  int kstar = 0;
  while (((int64_t)1 << (kstar + 1)) < L) ++kstar;
  return N < kstar ? N : kstar;
}

static int pick_group(int64_t ntiles, int64_t seqs, int want) {
  int g = want;
  while (g > 1 && ceil_div(ntiles, g) * seqs < 2 * 148) g /= 2;
  return g;
}

int engine_bank_tc(int n, int m, int64_t L, int batch, const int* N_host, int N_max, const void* pack,
                   const double* Bbar, const double* C, const double* D, const void* u, void* y, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  BankWs w = carve_bank(ws, n, m, L, batch);
  if (ws_bytes < w.bytes) return CASC_ERR_WORKSPACE;
  PackLayout P = pack_layout(const_cast<void*>(pack), n, m, N_max, CASC_FP32);
  const int64_t mm = (int64_t)m * m;
  int rc;

  std::vector<int> meta((size_t)4 * n);
  int *Neff = meta.data(), *Kc = Neff + n, *par = Neff + 2 * n, *order = Neff + 3 * n;
  int maxNe = 0;
  for (int s = 0; s < n; ++s) {
    Neff[s] = eff_order_b(N_host[s], L);
    Kc[s] = std::min(kHeadK, Neff[s]);
    par[s] = (Neff[s] - Kc[s]) % 2;
    maxNe = std::max(maxNe, Neff[s]);
  }
  std::iota(order, order + n, 0);
  std::stable_sort(order, order + n, [&](int a, int b) { return Neff[a] > Neff[b]; });
  CASC_TRY(cudaMemcpyAsync(w.meta, meta.data(), meta.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  const int *dNeff = w.meta, *dKc = w.meta + n, *dpar = w.meta + 2 * n, *dorder = w.meta + 3 * n;

  // ---- derived: Krylov columns, w = C P_Ne, fp32 copies
  {
    ProfScope ps(st, K_DERIVED, 0.0, 2.0 * n * (double)m * m * 128);
    if ((rc = launch_kr_init(Bbar, w.Kr64, n, m, st))) return rc;
    const int maxKc = std::min(kHeadK, maxNe);
    for (int i = 0; i < maxKc; ++i) {          // Kr[:, 2^i + j] = P_i Kr[:, j], j < 2^i
      DgemmArg a{};
      a.M = m; a.N = 1 << i; a.K = m;
      a.A = P.p64 + i * mm; a.lda = m; a.sA = (int64_t)(N_max + 1) * mm;
      a.B = w.Kr64; a.ldb = 128; a.sB = (int64_t)m * 128;
      a.C = w.Kr64 + (1 << i); a.ldc = 128; a.sC = (int64_t)m * 128;
      a.skip_below = dKc; a.level = i + 1;
      if ((rc = launch_dgemm(a, n, st))) return rc;
    }
    if ((rc = launch_kr_split(w.Kr64, dKc, w.krT, n, m, st))) return rc;
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
  const int64_t ntiles = ceil_div(L, 128);
  // ---- head: stages 0..Kc-1 (+ Bbar u), all channels
  {
    BankHeadArg a{};
    a.u = static_cast<const float*>(u); a.krT = w.krT; a.V = static_cast<float*>(w.Va);
    a.sys_list = dorder; a.n_list = n; a.L = L; a.batch = batch;
    a.tiles_per_cta = pick_group(ntiles, (int64_t)n * batch, 16);
    ProfScope ps(st, K_BANK_HEAD, (double)n * batch * L * (1 + m) * 4.0,
                 (double)n * batch * L * 2.0 * m * 128);
    if ((rc = launch_bank_head(m, a, st))) return rc;
  }
  // ---- streaming stages k >= kHeadK over the channels with Neff > k (a prefix of `order`)
  for (int k = kHeadK; k < maxNe; ++k) {
    int cnt = 0;
    while (cnt < n && Neff[order[cnt]] > k) ++cnt;
    BankStageArg a{};
    const int j = k - kHeadK;
    a.Vs = static_cast<const float*>(j % 2 == 0 ? w.Va : w.Vb);
    a.Vd = static_cast<float*>(j % 2 == 0 ? w.Vb : w.Va);
    a.P = P.f32; a.k = k; a.slots = N_max + 1;
    a.copy_from = (k == kHeadK) ? 0 : ((int64_t)1 << (k - 1));
    a.sys_list = dorder; a.n_list = cnt; a.L = L; a.batch = batch;
    a.tiles_per_cta = pick_group(ntiles, (int64_t)cnt * batch, 8);
    ProfScope ps(st, K_BANK_STAGE, 2.0 * cnt * batch * L * m * 4.0, 2.0 * cnt * batch * L * (double)mm);
    // Kernel choice (CASC_BANK_STAGE for A/B measurements): the TMA-pipelined shifted GEMM
    // (mimo_tc.cu, 3xTF32, per-channel weight planes) for m % 64 == 0, else the
    // register-prefetch kernel; "rp" / "ws" force the older variants.
    static const char mode_env = [] {
      const char* e = getenv("CASC_BANK_STAGE");
      return e ? e[0] : 't';
    }();
    if (mode_env == 'w') {
      rc = launch_bank_stage_ws(m, a, st);
    } else if (mode_env == 'r' || m % 64 != 0) {
      rc = launch_bank_stage_rp(m, a, st);
    } else {
      MimoGemm g{};
      g.src[0].A = a.Vs; g.src[0].W = P.f32; g.src[0].K = m; g.src[0].shift = (int64_t)1 << k;
      g.src[0].w_plane_off = 2 * k; g.src[0].w_planes = (int64_t)n * (N_max + 1) * 2;
      g.n_src = 1; g.R = a.Vs; g.out = a.Vd; g.n_out = m; g.L = L; g.batch = batch;
      g.sys_list = dorder; g.n_list = cnt; g.n_sys_total = n;
      g.w_plane_stride = 2 * (N_max + 1); g.t_first = (int)(a.copy_from / 128);
      rc = launch_mimo_gemm(g, true, st);
    }
    if (rc) return rc;
  }
  // ---- tail: stage Ne + y = C v + D u
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
