// C ABI of libcascade_b200 (declared in include/cascade.h) and the host-side engine that
// sequences the kernels of the cascade on one stream.
//
// Step schedule for system s with effective order Ne = min(N_s, floor(log2(L-1))) (stages with
// 2^k >= L are identities, R20):
//   derived   (fp64)   Abar Bbar, C P_Ne, C Bbar + D, C Abar Bbar              (tiny GEMMs)
//   first     (a2)     v^(1)_l = Bbar u_l + Abar Bbar u_{l-1}        = stages "B u" and k = 0
//   stage k   (a4)     v^(k+1)_l = v^(k)_l + P_k v^(k)_{l-2^k}           k = 1 .. Ne-1
//   last      (a5)     y_l = C v_l + (C P_Ne) v_{l-2^Ne} + D u_l           = stage Ne and y
//   Ne == 0            y_l = (C Bbar + D) u_l + C Abar Bbar u_{l-1}      (one kernel)
// The fused first/last forms are exact regroupings of PAPER.md:187 / :217-228 (associativity;
// DESIGN.md R21). v^(k) ping-pongs between two workspace buffers: after stage k it sits in
// buffer k % 2.
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <numeric>

#include "common.cuh"
#include "kernels.cuh"
#include "engine.cuh"
#include "profile.cuh"

namespace casc {

thread_local int g_launches = 0;

struct ApplyWs {
  int* meta;                        // Neff | order | direct | groupA | groupB   (5 n ints)
  double *AB64, *CP64, *CBD64, *CAB64;
  float *Bb32, *AB32, *C32, *CP32, *D32, *CBD32, *CAB32;
  void *Va, *Vb;
  size_t bytes;
};

static ApplyWs carve_apply(void* ws, int n, int m, int p, int q, int64_t L, int batch, int mode) {
  Carver c(ws);
  ApplyWs w{};
  const size_t es = (mode == CASC_BF16) ? 2 : 4;
  w.meta = c.take<int>((size_t)5 * n);
  w.AB64 = c.take<double>((size_t)n * m * p);
  w.CP64 = c.take<double>((size_t)n * q * m);
  w.CBD64 = c.take<double>((size_t)n * q * p);
  w.CAB64 = c.take<double>((size_t)n * q * p);
  w.Bb32 = c.take<float>((size_t)n * m * p);
  w.AB32 = c.take<float>((size_t)n * m * p);
  w.C32 = c.take<float>((size_t)n * q * m);
  w.CP32 = c.take<float>((size_t)n * q * m);
  w.D32 = c.take<float>((size_t)n * q * p);
  w.CBD32 = c.take<float>((size_t)n * q * p);
  w.CAB32 = c.take<float>((size_t)n * q * p);
  const size_t vbytes = (size_t)n * batch * (size_t)L * m * es;
  w.Va = c.take<char>(vbytes);
  w.Vb = c.take<char>(vbytes);
  w.bytes = c.bytes();
  return w;
}

// bf16 SISO banks (bf16 storage of u and y) run the fp32 tensor-core bank path on fp32 copies of
// u and y carved in front of its workspace: the arithmetic is the fp32 path's (3xTF32, at least
// the bf16 mode's fp32 accumulation), y is rounded once to bf16 (RN-even)
static bool bank_bf16_path(int m, int p, int q, int mode) {
  return mode == CASC_BF16 && bank_tc_path(m, p, q, CASC_FP32);
}
__global__ void bf16_to_f32_kernel(const __nv_bfloat16* src, float* dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __bfloat162float(src[i]);
}
__global__ void f32_to_bf16_kernel(const float* src, __nv_bfloat16* dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

size_t apply_ws_bytes(int n, int m, int p, int q, int64_t L, int batch, int mode, int n_max) {
  if (bank_tc_path(m, p, q, mode)) return bank_ws_bytes(n, m, L, batch, n_max);
  if (bank_bf16_path(m, p, q, mode))
    return align_up((size_t)2 * n * batch * L * sizeof(float), 256) + bank_ws_bytes(n, m, L, batch, n_max);
  if (mimo_tc_path(n, m, p, q, mode)) return mimo_ws_bytes(m, p, q, L, batch, mode);
  return carve_apply(nullptr, n, m, p, q, L, batch, mode).bytes;
}

int validate_common(int n, int m, int p, int q, int64_t L, int batch, int N_max, int mode) {
  if (n < 0 || m < 1 || p < 1 || q < 1 || L < 0 || batch < 0 || N_max < 0) return CASC_ERR_ARG;
  if (mode != CASC_FP32 && mode != CASC_BF16) return CASC_ERR_ARG;
  if (p > m || q > m) return CASC_ERR_DIM;
  if (N_max > 62) return CASC_ERR_DIM;
  if (m > 4096) return CASC_ERR_UNSUPPORTED;
  if (n == 0 || L == 0 || batch == 0) return kEmptyCall;   // nothing to compute, no buffer touched
  return CASC_OK;
}

// The engine: n systems sharing (m, p, q), per-system N_host[s].
int engine_apply(int n, int m, int p, int q, int64_t L, int batch, const int* N_host, int N_max,
                 int mode, const void* pack, const double* Bbar, const double* C, const double* D,
                 const void* u, void* y, void* ws, size_t ws_bytes, cudaStream_t st) {
  int rc = validate_common(n, m, p, q, L, batch, N_max, mode);
  if (rc == kEmptyCall) return CASC_OK;
  if (rc) return rc;
  if (!N_host || !pack || !Bbar || !C || !u || !y || !ws) return CASC_ERR_ARG;
  for (int s = 0; s < n; ++s)
    if (N_host[s] < 0 || N_host[s] > N_max) return CASC_ERR_DIM;
  if (bank_tc_path(m, p, q, mode))
    return engine_bank_tc(n, m, L, batch, N_host, N_max, pack, Bbar, C, D, u, y, ws, ws_bytes, st);
  if (bank_bf16_path(m, p, q, mode)) {
    const int64_t cnt = (int64_t)n * batch * L;
    const size_t front = align_up((size_t)2 * cnt * sizeof(float), 256);
    if (ws_bytes <= front) return CASC_ERR_WORKSPACE;
    float* u32 = static_cast<float*>(ws);
    float* y32 = u32 + cnt;
    const int blocks = (int)std::min<int64_t>(ceil_div(cnt, 256), 148 * 8);
    bf16_to_f32_kernel<<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(u), u32, cnt);
    CASC_LAUNCHED();
    // the bf16 pack of a bank-sized system also holds the tf32 planes (common.cuh pack_layout)
    int rc2 = engine_bank_tc(n, m, L, batch, N_host, N_max, pack, Bbar, C, D, u32, y32, (char*)ws + front,
                             ws_bytes - front, st);
    if (rc2) return rc2;
    f32_to_bf16_kernel<<<blocks, 256, 0, st>>>(y32, static_cast<__nv_bfloat16*>(y), cnt);
    CASC_LAUNCHED();
    return CASC_OK;
  }
  if (mimo_tc_path(n, m, p, q, mode))
    return engine_mimo_tc(m, p, q, L, batch, N_host[0], N_max, mode, pack, Bbar, C, D, u, y, ws, ws_bytes, st);
  ApplyWs w = carve_apply(ws, n, m, p, q, L, batch, mode);
  if (ws_bytes < w.bytes) return CASC_ERR_WORKSPACE;
  PackLayout P = pack_layout(const_cast<void*>(pack), n, m, N_max, mode);
  const bool bf = (mode == CASC_BF16);
  const int64_t mm = (int64_t)m * m;
  const double es = bf ? 2.0 : 4.0;

  // ---- host metadata: effective orders and launch lists
  std::vector<int> meta((size_t)5 * n);
  int* Neff = meta.data();
  int *order = Neff + n, *direct = Neff + 2 * n, *gA = Neff + 3 * n, *gB = Neff + 4 * n;
  int maxNe = 0;
  for (int s = 0; s < n; ++s) {
    Neff[s] = eff_order(N_host[s], L);
    maxNe = std::max(maxNe, Neff[s]);
  }
  int n1 = 0, n0 = 0, na = 0, nb = 0;
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return Neff[a] > Neff[b]; });
  for (int s : idx) {
    if (Neff[s] >= 1) {
      order[n1++] = s;
      if ((Neff[s] - 1) % 2 == 0) gA[na++] = s; else gB[nb++] = s;
    } else {
      direct[n0++] = s;
    }
  }
  CASC_TRY(cudaMemcpyAsync(w.meta, meta.data(), meta.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  const int* dNeff = w.meta;
  const int *dorder = w.meta + n, *ddirect = w.meta + 2 * n, *dgA = w.meta + 3 * n, *dgB = w.meta + 4 * n;

  // ---- derived float64 matrices (tiny)
  {
    ProfScope ps(st, K_DERIVED, 0.0, 2.0 * n * ((double)m * m * p + (double)q * m * m + 2.0 * q * m * p));
    DgemmArg a{};
    // AB = P_0 Bbar  (m x p)
    a = DgemmArg{};
    a.M = m; a.N = p; a.K = m;
    a.A = P.p64; a.lda = m; a.sA = (N_max + 1) * mm;
    a.B = Bbar; a.ldb = p; a.sB = (int64_t)m * p;
    a.C = w.AB64; a.ldc = p; a.sC = (int64_t)m * p;
    if ((rc = launch_dgemm(a, n, st))) return rc;
    // CP = C P_Ne  (q x m)
    a = DgemmArg{};
    a.M = q; a.N = m; a.K = m;
    a.A = C; a.lda = m; a.sA = (int64_t)q * m;
    a.B = P.p64; a.ldb = m; a.sB = (N_max + 1) * mm; a.nB = mm; a.selB = dNeff;
    a.C = w.CP64; a.ldc = m; a.sC = (int64_t)q * m;
    if ((rc = launch_dgemm(a, n, st))) return rc;
    // CBD = C Bbar + D  (q x p)
    a = DgemmArg{};
    a.M = q; a.N = p; a.K = m;
    a.A = C; a.lda = m; a.sA = (int64_t)q * m;
    a.B = Bbar; a.ldb = p; a.sB = (int64_t)m * p;
    a.C = w.CBD64; a.ldc = p; a.sC = (int64_t)q * p;
    a.Cadd = D; a.sCadd = (int64_t)q * p;
    if ((rc = launch_dgemm(a, n, st))) return rc;
    // CAB = C (Abar Bbar)  (q x p)
    a = DgemmArg{};
    a.M = q; a.N = p; a.K = m;
    a.A = C; a.lda = m; a.sA = (int64_t)q * m;
    a.B = w.AB64; a.ldb = p; a.sB = (int64_t)m * p;
    a.C = w.CAB64; a.ldc = p; a.sC = (int64_t)q * p;
    if ((rc = launch_dgemm(a, n, st))) return rc;
  }
  {
  ProfScope ps(st, K_CONVERT, 0.0, 0.0);
  if ((rc = launch_f64_to_f32(Bbar, w.Bb32, (int64_t)n * m * p, st))) return rc;
  if ((rc = launch_f64_to_f32(w.AB64, w.AB32, (int64_t)n * m * p, st))) return rc;
  if ((rc = launch_f64_to_f32(C, w.C32, (int64_t)n * q * m, st))) return rc;
  if ((rc = launch_f64_to_f32(w.CP64, w.CP32, (int64_t)n * q * m, st))) return rc;
  if ((rc = launch_f64_to_f32(w.CBD64, w.CBD32, (int64_t)n * q * p, st))) return rc;
  if ((rc = launch_f64_to_f32(w.CAB64, w.CAB32, (int64_t)n * q * p, st))) return rc;
  if (D) {
    if ((rc = launch_f64_to_f32(D, w.D32, (int64_t)n * q * p, st))) return rc;
  } else {
    CASC_TRY(cudaMemsetAsync(w.D32, 0, sizeof(float) * (size_t)n * q * p, st));
  }
  }

  const int64_t u_sys = (int64_t)batch * L * p, y_sys = (int64_t)batch * L * q;
  const int64_t v_sys = (int64_t)batch * L * m;
  auto base = [&](GemmArg& g) {
    g = GemmArg{};
    g.L = L; g.batch = batch; g.Neff = dNeff;
  };
  auto src = [&](SrcArg& sa, const void* A, int64_t A_sys, int K, const void* W, int64_t W_sys,
                 int w_bf16, const float* Wlo, int64_t shift, int from_N) {
    sa.A = A; sa.A_sys = A_sys; sa.K = K; sa.a_bf16 = bf;
    sa.W = W; sa.W_sys = W_sys; sa.w_bf16 = w_bf16; sa.Wlo = Wlo;
    sa.shift = shift; sa.shift_from_N = from_N;
  };

  // ---- Ne == 0 systems: y = (C Bbar + D) u_l + (C Abar Bbar) u_{l-1}
  if (n0 > 0) {
    GemmArg g; base(g);
    src(g.src[0], u, u_sys, p, w.CBD32, (int64_t)q * p, 0, nullptr, 0, 0);
    src(g.src[1], u, u_sys, p, w.CAB32, (int64_t)q * p, 0, nullptr, 1, 0);
    g.n_src = 2;
    g.out = y; g.out_sys = y_sys; g.out_bf16 = bf; g.n_out = q;
    g.sys_list = ddirect; g.n_list = n0;
    ProfScope ps(st, K_DIRECT, (double)n0 * batch * L * (p + q) * es, (double)n0 * batch * L * 4.0 * q * p);
    if ((rc = launch_simt_gemm(g, st))) return rc;
  }
  if (n1 == 0) return CASC_OK;

  // ---- first (a2): v^(1) = Bbar u_l + Abar Bbar u_{l-1}  -> Va
  {
    GemmArg g; base(g);
    src(g.src[0], u, u_sys, p, w.Bb32, (int64_t)m * p, 0, nullptr, 0, 0);
    src(g.src[1], u, u_sys, p, w.AB32, (int64_t)m * p, 0, nullptr, 1, 0);
    g.n_src = 2;
    g.out = w.Va; g.out_sys = v_sys; g.out_bf16 = bf; g.n_out = m;
    g.sys_list = dorder; g.n_list = n1;
    ProfScope ps(st, K_FIRST, (double)n1 * batch * L * (p + m) * es, (double)n1 * batch * L * 4.0 * m * p);
    if ((rc = launch_simt_gemm(g, st))) return rc;
  }
  // ---- stages k = 1 .. maxNe-1 (a4) over the systems with Neff >= k+1 (a prefix of order)
  for (int k = 1; k <= maxNe - 1; ++k) {
    int cnt = 0;
    while (cnt < n1 && Neff[order[cnt]] >= k + 1) ++cnt;
    void* Vs = (k - 1) % 2 == 0 ? w.Va : w.Vb;
    void* Vd = (k % 2 == 0) ? w.Va : w.Vb;
    GemmArg g; base(g);
    if (bf) {
      src(g.src[0], Vs, v_sys, m, P.b16 + k * mm, (N_max + 1) * mm, 1, nullptr, (int64_t)1 << k, 0);
    } else {
      const float* hi = P.f32 + (int64_t)k * 2 * mm;
      src(g.src[0], Vs, v_sys, m, hi, (N_max + 1) * 2 * mm, 0, hi + mm, (int64_t)1 << k, 0);
    }
    g.n_src = 1;
    g.R = Vs; g.R_sys = v_sys;
    g.out = Vd; g.out_sys = v_sys; g.out_bf16 = bf; g.n_out = m;
    g.sys_list = dorder; g.n_list = cnt;
    ProfScope ps(st, K_STAGE, 2.0 * cnt * batch * L * m * es, 2.0 * cnt * batch * L * (double)m * m);
    if ((rc = launch_simt_gemm(g, st))) return rc;
  }
  // ---- last (a5): y = C v + (C P_Ne) v_{l-2^Ne} + D u, per buffer parity group
  for (int grp = 0; grp < 2; ++grp) {
    const int cnt = grp == 0 ? na : nb;
    if (cnt == 0) continue;
    void* V = grp == 0 ? w.Va : w.Vb;
    GemmArg g; base(g);
    src(g.src[0], V, v_sys, m, w.C32, (int64_t)q * m, 0, nullptr, 0, 0);
    src(g.src[1], V, v_sys, m, w.CP32, (int64_t)q * m, 0, nullptr, 0, 1);
    src(g.src[2], u, u_sys, p, w.D32, (int64_t)q * p, 0, nullptr, 0, 0);
    g.n_src = D ? 3 : 2;
    g.out = y; g.out_sys = y_sys; g.out_bf16 = bf; g.n_out = q;
    g.sys_list = grp == 0 ? dgA : dgB; g.n_list = cnt;
    ProfScope ps(st, K_LAST, (double)cnt * batch * L * (m + p + q) * es,
                 (double)cnt * batch * L * (4.0 * q * m + 2.0 * q * p));
    if ((rc = launch_simt_gemm(g, st))) return rc;
  }
  return CASC_OK;
}

int DevCtx::ensure_pinned(size_t n_ints) {
  if (pinned_n >= n_ints) return CASC_OK;
  if (pinned) cudaFreeHost(pinned);
  pinned = nullptr;
  pinned_n = 0;
  CASC_TRY(cudaHostAlloc(&pinned, sizeof(int) * n_ints, cudaHostAllocDefault));
  pinned_n = n_ints;
  return CASC_OK;
}

int DevCtx::ensure_dmeta(size_t n_ints) {
  if (dmeta_n >= n_ints) return CASC_OK;
  if (dmeta) cudaFree(dmeta);
  dmeta = nullptr;
  dmeta_n = 0;
  CASC_TRY(cudaMalloc(&dmeta, sizeof(int) * n_ints));
  dmeta_n = n_ints;
  return CASC_OK;
}

DevCtx* dev_ctx() {
  static std::mutex create_mu;
  static DevCtx* ctx[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(create_mu);
  if (!ctx[dev]) {
    DevCtx* c = new DevCtx();
    if (cudaStreamCreateWithFlags(&c->in, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->out, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->inputs_free, cudaEventDisableTiming) != cudaSuccess)
      return nullptr;
    ctx[dev] = c;
  }
  return ctx[dev];
}

static int coop_max_m() {                          // diagnostics A/B: CASC_POWERS_COOP_MAX
  static const int v = [] {
    const char* e = getenv("CASC_POWERS_COOP_MAX");
    return e ? atoi(e) : 512;
  }();
  return v;
}
int engine_powers(int n, int m, const int* N_host, int N_max, const double* Abar, int mode,
                  void* pack, cudaStream_t st) {
  if (n < 0 || m < 1 || N_max < 0) return CASC_ERR_ARG;
  if (mode != CASC_FP32 && mode != CASC_BF16) return CASC_ERR_ARG;
  if (N_max > 62) return CASC_ERR_DIM;
  if (m > 4096) return CASC_ERR_UNSUPPORTED;
  if (n == 0) return CASC_OK;                       // no systems: nothing to compute
  if (!N_host || !Abar || !pack) return CASC_ERR_ARG;
  for (int s = 0; s < n; ++s)
    if (N_host[s] < 0 || N_host[s] > N_max) return CASC_ERR_DIM;
  PackLayout P = pack_layout(pack, n, m, N_max, mode);
  const int64_t mm = (int64_t)m * m, sys = (N_max + 1) * mm;
  CASC_TRY(cudaMemcpyAsync(P.hdr, N_host, sizeof(int) * n, cudaMemcpyHostToDevice, st));
  if (m <= 64) {                                  // banks: all squarings + packing in one launch
    int maxN = *std::max_element(N_host, N_host + n);
    ProfScope ps(st, K_POWERS, 16.0 * n * mm * (maxN + 1), 2.0 * n * (double)mm * m * maxN);
    ps.exec(16.0 * n * mm * (maxN + 1), 2.0 * n * (double)mm * m * maxN, PIPE_FP64);
    return launch_powers_small(P, Abar, n, N_max, m, st);
  }
  // MIMO with m <= 512: one cooperative launch (squarings + pack); E3 powers 0.38 -> 0.28 ms. At
  // m = 1024 (256 tiles per level) the per-level launches measured faster (E4: 2.08 vs 2.39 ms, A/B)
  if (n == 1 && m <= coop_max_m()) {
    ProfScope ps(st, K_POWERS, 16.0 * mm * (N_host[0] + 1), 2.0 * (double)mm * m * N_host[0]);
    ps.exec(24.0 * mm * N_host[0] + 16.0 * mm * (N_host[0] + 1), 2.0 * (double)mm * m * N_host[0], PIPE_FP64);
    return launch_powers_coop(P, Abar, N_host[0], m, st);
  }
  // P_0 = Abar (strided copy into slot 0 of every system)
  CASC_TRY(cudaMemcpy2DAsync(P.p64, sys * sizeof(double), Abar, mm * sizeof(double),
                             mm * sizeof(double), n, cudaMemcpyDeviceToDevice, st));
  int maxN = *std::max_element(N_host, N_host + n);
  for (int k = 1; k <= maxN; ++k) {               // P_k = P_{k-1} P_{k-1}
    int cnt = 0;
    for (int s = 0; s < n; ++s) cnt += N_host[s] >= k;
    ProfScope ps(st, K_POWERS, 16.0 * cnt * mm, 2.0 * cnt * (double)mm * m);
    ps.exec(24.0 * cnt * mm, 2.0 * cnt * (double)mm * m, PIPE_FP64);
    DgemmArg a{};
    a.M = m; a.N = m; a.K = m;
    a.A = P.p64 + (k - 1) * mm; a.lda = m; a.sA = sys;
    a.B = P.p64 + (k - 1) * mm; a.ldb = m; a.sB = sys;
    a.C = P.p64 + k * mm; a.ldc = m; a.sC = sys;
    a.skip_below = P.hdr; a.level = k;
    int rc = launch_dgemm(a, n, st);
    if (rc) return rc;
  }
  ProfScope ps(st, K_PACK, 0.0, 0.0);
  return launch_pack(P, n, N_max, m, st);
}

}  // namespace casc

using namespace casc;

extern "C" {

const char* casc_status_str(int s) {
  switch (s) {
    case CASC_OK: return "CASC_OK";
    case CASC_ERR_ARG: return "CASC_ERR_ARG";
    case CASC_ERR_DIM: return "CASC_ERR_DIM";
    case CASC_ERR_NONSQUARE: return "CASC_ERR_NONSQUARE";
    case CASC_ERR_UNSUPPORTED: return "CASC_ERR_UNSUPPORTED";
    case CASC_ERR_WORKSPACE: return "CASC_ERR_WORKSPACE";
    case CASC_ERR_CUDA: return "CASC_ERR_CUDA";
    case CASC_ERR_NCCL: return "CASC_ERR_NCCL";
    default: return "CASC_ERR_UNKNOWN";
  }
}

int casc_version(void) { return 100; }
int casc_target_sm(void) { return 100; }
int casc_last_launch_count(void) { return g_launches; }

size_t casc_pack_bytes(int n_sys, int m, int N_max, int mode) {
  if (n_sys < 1 || m < 1 || N_max < 0) return 0;
  return pack_layout(nullptr, n_sys, m, N_max, mode).bytes;
}

int casc_powers(int n_sys, int m, const int* N_host, int N_max, const double* Abar, int mode,
                void* pack, void* stream) {
  g_launches = 0;
  return engine_powers(n_sys, m, N_host, N_max, Abar, mode, pack, (cudaStream_t)stream);
}

int casc_powers_norms(int n_sys, int m, int N_max, int mode, const void* pack, double* norms_host, void* stream) {
  g_launches = 0;
  if (n_sys < 1 || m < 1 || N_max < 0 || !pack || !norms_host) return CASC_ERR_ARG;
  if (mode != CASC_FP32 && mode != CASC_BF16) return CASC_ERR_ARG;
  if (N_max > 62) return CASC_ERR_DIM;
  cudaStream_t st = (cudaStream_t)stream;
  DevCtx* ctx = dev_ctx();
  if (!ctx) return CASC_ERR_CUDA;
  std::lock_guard<std::mutex> lock(ctx->mu);
  const size_t n = (size_t)n_sys * (N_max + 2);
  if (ctx->dnorm_n < n) {
    if (ctx->dnorm) cudaFree(ctx->dnorm);
    ctx->dnorm = nullptr;
    ctx->dnorm_n = 0;
    CASC_TRY(cudaMalloc(&ctx->dnorm, n * sizeof(double)));
    ctx->dnorm_n = n;
  }
  PackLayout P = pack_layout(const_cast<void*>(pack), n_sys, m, N_max, mode);
  std::vector<int> Ns(n_sys);
  CASC_TRY(cudaMemsetAsync(ctx->dnorm, 0, n * sizeof(double), st));
  CASC_TRY(cudaMemcpyAsync(Ns.data(), P.hdr, sizeof(int) * n_sys, cudaMemcpyDeviceToHost, st));
  int rc = launch_powers_sumsq(P, n_sys, N_max, m, ctx->dnorm, st);
  if (rc) return rc;
  CASC_TRY(cudaMemcpyAsync(norms_host, ctx->dnorm, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  CASC_TRY(cudaStreamSynchronize(st));
  for (int s = 0; s < n_sys; ++s)
    for (int k = 0; k < N_max + 2; ++k) {
      double& v = norms_host[(size_t)s * (N_max + 2) + k];
      v = k <= Ns[s] + 1 ? sqrt(v) : NAN;
    }
  return CASC_OK;
}

size_t casc_apply_workspace_bytes(int m, int p, int q, int64_t L, int batch, int N, int mode) {

  if (m < 1 || p < 1 || q < 1 || L < 1 || batch < 1) return 0;
  return apply_ws_bytes(1, m, p, q, L, batch, mode, N);
}

int casc_apply(int m, int p, int q, int64_t L, int batch, int N, int N_max, int mode,
               const void* pack, const double* Bbar, const double* C, const double* D,
               const void* u, void* y, void* ws, size_t ws_bytes, int* effective_stages,
               void* stream) {
  g_launches = 0;
  if (N < 0) return CASC_ERR_ARG;
  int rc = engine_apply(1, m, p, q, L, batch, &N, N_max, mode, pack, Bbar, C, D, u, y, ws,
                        ws_bytes, (cudaStream_t)stream);
  if (rc == CASC_OK && effective_stages) {
    int e = 0;
    for (int k = 0; k <= N; ++k)
      if (((int64_t)1 << k) < L) ++e;
    *effective_stages = e;
  }
  return rc;
}

size_t casc_bank_workspace_bytes(int n_ch, int m, int64_t L, int batch, int N_max, int mode) {

  if (n_ch < 1 || m < 1 || L < 1 || batch < 1) return 0;
  return apply_ws_bytes(n_ch, m, 1, 1, L, batch, mode, N_max);
}

int casc_apply_bank(int n_ch, int m, int64_t L, int batch, const int* N_host, int N_max,
                    int mode, const void* pack, const double* Bbar, const double* C,
                    const double* D, const void* u, void* y, void* ws, size_t ws_bytes,
                    void* stream) {
  g_launches = 0;
  return engine_apply(n_ch, m, 1, 1, L, batch, N_host, N_max, mode, pack, Bbar, C, D, u, y, ws,
                      ws_bytes, (cudaStream_t)stream);
}

struct HostWs {
  double *Abar, *Bbar, *C, *D;
  void *u, *y, *pack, *apply_ws;
  size_t apply_bytes, bytes;
};

static HostWs carve_host(void* base, int n, int m, int p, int q, int64_t L, int batch, int N_max,
                         int mode) {
  Carver c(base);
  HostWs h{};
  const size_t es = (mode == CASC_BF16) ? 2 : 4;
  h.Abar = c.take<double>((size_t)n * m * m);
  h.Bbar = c.take<double>((size_t)n * m * p);
  h.C = c.take<double>((size_t)n * q * m);
  h.D = c.take<double>((size_t)n * q * p);
  h.u = c.take<char>((size_t)n * batch * L * p * es);
  h.y = c.take<char>((size_t)n * batch * L * q * es);
  h.pack = c.take<char>(pack_layout(nullptr, n, m, N_max, mode).bytes);
  h.apply_bytes = apply_ws_bytes(n, m, p, q, L, batch, mode, N_max);
  h.apply_ws = c.take<char>(h.apply_bytes);
  h.bytes = c.bytes();
  return h;
}

size_t casc_run_host_bytes(int n_sys, int m, int p, int q, int64_t L, int batch, int N_max,
                           int mode) {
  if (n_sys < 1 || m < 1 || p < 1 || q < 1 || L < 1 || batch < 1 || N_max < 0) return 0;
  return carve_host(nullptr, n_sys, m, p, q, L, batch, N_max, mode).bytes;
}

int casc_run_host(int n_sys, int m, int p, int q, int64_t L, int batch, const int* N_host,
                  int N_max, int mode, const double* Abar_h, const double* Bbar_h,
                  const double* C_h, const double* D_h, const void* u_h, void* y_h,
                  void* dev_ws, size_t dev_ws_bytes, void* stream) {
  int rc = validate_common(n_sys, m, p, q, L, batch, N_max, mode);
  if (rc == kEmptyCall) return CASC_OK;
  if (rc) return rc;
  if (!N_host || !Abar_h || !Bbar_h || !C_h || !u_h || !y_h || !dev_ws) return CASC_ERR_ARG;
  if (n_sys > 1 && (p != 1 || q != 1)) return CASC_ERR_UNSUPPORTED;
  HostWs h = carve_host(dev_ws, n_sys, m, p, q, L, batch, N_max, mode);
  // the apply workspace is the last region: a smaller dev_ws leaves it short, which banks absorb
  // by running in channel waves (engine_apply reports CASC_ERR_WORKSPACE otherwise)
  const size_t fixed = (size_t)((char*)h.apply_ws - (char*)dev_ws);
  if (dev_ws_bytes <= fixed) {
    if (getenv("CASC_DEBUG")) fprintf(stderr, "casc: run_host ws=%zu fixed=%zu\n", dev_ws_bytes, fixed);
    return CASC_ERR_WORKSPACE;
  }
  h.apply_bytes = std::min(h.apply_bytes, dev_ws_bytes - fixed);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t es = (mode == CASC_BF16) ? 2 : 4;
  DevCtx* ctx = dev_ctx();
  if (!ctx) return CASC_ERR_CUDA;
  // calls on one device share the context's copy streams and pinned staging: serialise them
  std::lock_guard<std::mutex> lock(ctx->mu);
  if (n_sys > 1 && m == 64 && bank_tc_path(m, p, q, mode)) {
    // banks: parameters and powers on `st`; each wave's u arrives on the copy-in stream and
    // finished channels' outputs go back while later stage passes run
    for (int s = 0; s < n_sys; ++s)
      if (N_host[s] < 0 || N_host[s] > N_max) return CASC_ERR_DIM;
    if (getenv("CASC_TIMING")) {                        // diagnostics: timeline origin (bank_engine.cu)
      if (!casc::g_timing_t0) cudaEventCreate(&casc::g_timing_t0);
      cudaEventRecord(casc::g_timing_t0, st);
    }
    CASC_TRY(cudaMemcpyAsync(h.Abar, Abar_h, sizeof(double) * n_sys * m * m, cudaMemcpyHostToDevice, st));
    CASC_TRY(cudaMemcpyAsync(h.Bbar, Bbar_h, sizeof(double) * n_sys * m, cudaMemcpyHostToDevice, st));
    CASC_TRY(cudaMemcpyAsync(h.C, C_h, sizeof(double) * n_sys * m, cudaMemcpyHostToDevice, st));
    if (D_h) CASC_TRY(cudaMemcpyAsync(h.D, D_h, sizeof(double) * n_sys, cudaMemcpyHostToDevice, st));
    CASC_TRY(cudaEventRecord(ctx->inputs_free, st));   // the first wave's input copy overlaps the powers
    rc = engine_powers(n_sys, m, N_host, N_max, h.Abar, mode, h.pack, st);
    if (rc) return rc;
    rc = engine_bank_pipelined(n_sys, m, L, batch, N_host, N_max, h.pack, h.Bbar, h.C, D_h ? h.D : nullptr,
                               static_cast<float*>(h.u), static_cast<float*>(h.y), u_h, y_h, h.apply_ws,
                               h.apply_bytes, st, ctx);
    // else the serial path below (e.g. CASC_BANK_AB=0, which has no per-channel output streaming)
    if (rc != CASC_ERR_WORKSPACE && rc != CASC_ERR_UNSUPPORTED) return rc;
  }
  CASC_TRY(cudaMemcpyAsync(h.Abar, Abar_h, sizeof(double) * n_sys * m * m, cudaMemcpyHostToDevice, st));
  CASC_TRY(cudaMemcpyAsync(h.Bbar, Bbar_h, sizeof(double) * n_sys * m * p, cudaMemcpyHostToDevice, st));
  CASC_TRY(cudaMemcpyAsync(h.C, C_h, sizeof(double) * n_sys * q * m, cudaMemcpyHostToDevice, st));
  if (D_h) CASC_TRY(cudaMemcpyAsync(h.D, D_h, sizeof(double) * n_sys * q * p, cudaMemcpyHostToDevice, st));
  if (n_sys == 1 && batch > 1 && mimo_tc_path(1, m, p, q, mode)) {
    // one MIMO system: the batch's sequences are independent, so they run in chunks whose input
    // copy (copy-in stream) overlaps the previous chunk's compute and whose output copy (copy-out
    // stream) overlaps the next chunk's; the input copy may start before the powers (they do not
    // touch u; E3: 0.67 ms of squarings)
    if (getenv("CASC_TIMING")) {                        // diagnostics: timeline origin
      if (!casc::g_timing_t0) cudaEventCreate(&casc::g_timing_t0);
      cudaEventRecord(casc::g_timing_t0, st);
    }
    CASC_TRY(cudaEventRecord(ctx->inputs_free, st));
    rc = engine_powers(1, m, N_host, N_max, h.Abar, mode, h.pack, st);
    if (rc) return rc;
    // batch chunks (CASC_MIMO_CHUNKS, tests): by default one per 64 MiB of input, 1..8 -- each chunk
    // adds its launches' fill/drain; the first input and last output chunk are exposed (E3 e2e: 4
    // chunks 14.8 ms, 8: 15.0, 16: 17.5; E4 with 4.3 GB of input takes 8)
    static const int chunks_env = [] {
      const char* e = getenv("CASC_MIMO_CHUNKS");
      return e ? std::max(1, atoi(e)) : 0;
    }();
    const int64_t in_bytes = (int64_t)es * batch * L * p;
    const int chunks = chunks_env ? chunks_env : (int)std::min<int64_t>(8, std::max<int64_t>(1, ceil_div(in_bytes, (int64_t)64 << 20)));
    // chunk boundaries: when chunks would hold several sequences, ramp up from and down to one
    // sequence (1, 2, 3, ..., 3, 2, 1): the exposed first input / last output copy is one sequence,
    // and each chunk's input (the copy is ~2x faster than the compute per sequence on E3) lands
    // while the previous chunk computes
    std::vector<int> sizes;
    if (chunks < batch && batch >= 4) {
      // arithmetic ramp 1, 2, 3, ... (E3 e2e: 1,2,3,4,3,2,1 9.72 ms vs the doubling 1,2,4,2,4,2,1 9.93)
      std::vector<int> up;
      int total = 0;
      for (int M = 1; 2 * (total + M) <= batch; ++M) { up.push_back(M); total += M; }
      sizes = up;
      for (int rest = batch - 2 * total; rest > 0;) { const int t = std::min(up.back() + 1, rest); sizes.push_back(t); rest -= t; }
      sizes.insert(sizes.end(), up.rbegin(), up.rend());
    } else {
      const int n0 = std::min(batch, chunks);
      for (int i = 0; i < n0; ++i) sizes.push_back((int)((int64_t)batch * (i + 1) / n0 - (int64_t)batch * i / n0));
    }
    if (const char* e = getenv("CASC_MIMO_SIZES")) {   // diagnostics A/B: explicit chunk sizes "1,3,4,..."
      std::vector<int> v;
      int tot = 0;
      for (const char* q = e; *q;) {
        const int x = atoi(q);
        if (x > 0) { v.push_back(x); tot += x; }
        while (*q && *q != ',') ++q;
        if (*q == ',') ++q;
      }
      if (tot == batch) sizes = v;
    }
    const int nc = (int)sizes.size();
    // derived weights once for all chunks (Ne is that of the full length L)
    const int Ne = eff_order(N_host[0], L);
    {
      MimoWs w = carve_mimo(h.apply_ws, m, p, q, L, batch, mode);
      if (h.apply_bytes < w.bytes) return CASC_ERR_WORKSPACE;
      PackLayout P = pack_layout(h.pack, 1, m, N_max, mode);
      if ((rc = mimo_derive(m, p, q, Ne, P, h.Bbar, h.C, D_h ? h.D : nullptr, w, mode == CASC_FP32, st))) return rc;
    }
    timing_mark("powers + derived", st);
    // The first and the last chunk are exposed (nothing to overlap their input / output copy with).
    // When such a chunk is a single sequence and the impulse response is short against L, it runs
    // as kW time windows (rows [r0, r1) computed from inputs [r0 - Hu, r1), Hu = 2^(Ne+1) - 1, exact:
    // PAPER.md:137-141, pin T14): the first chunk's compute starts after its first window's input
    // landed, the last chunk's output leaves window by window.
    static const int kW = [] {                        // windows per exposed chunk (CASC_MIMO_WINDOWS: diagnostics)
      const char* e = getenv("CASC_MIMO_WINDOWS");
      return e ? std::min(64, std::max(2, atoi(e))) : 8;
    }();
    const int64_t Hu = Ne > 0 ? ((int64_t)2 << Ne) - 1 : 0;
    const int64_t Lw = ceil_div(L, kW);
    std::vector<int> b0(nc + 1, 0);
    for (int i = 0; i < nc; ++i) b0[i + 1] = b0[i] + sizes[i];
    auto windowed = [&](int i) { return nc > 1 && (i == 0 || i == nc - 1) && b0[i + 1] - b0[i] == 1 && Ne > 0 && Lw >= 8 * Hu; };
    std::vector<cudaEvent_t> ev((size_t)2 * nc + 2 * kW, nullptr);
    for (auto& e : ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) { rc = CASC_ERR_CUDA; break; }
    cudaEvent_t* wev = ev.data() + 2 * nc;            // window events: inputs (first chunk), outputs (last)
    const size_t in_row = es * (size_t)L * p, out_row = es * (size_t)L * q;
    auto ok = [&](cudaError_t e) { if (e != cudaSuccess && rc == CASC_OK) rc = CASC_ERR_CUDA; return rc == CASC_OK; };
    auto win = [&](int j, int64_t* r0, int64_t* r1) { *r0 = std::min<int64_t>(L, j * Lw); *r1 = std::min<int64_t>(L, (j + 1) * Lw); };
    // chunk i+1's input is submitted after chunk i's work is queued: the small table upload inside
    // each chunk's apply queues behind every copy submitted before it on the copy engine
    auto submit = [&](int i) {
      if (i == 0 && windowed(0)) {                    // window by window
        for (int j = 0; j < kW; ++j) {
          int64_t r0, r1;
          win(j, &r0, &r1);
          if (!ok(cudaMemcpyAsync((char*)h.u + r0 * es * p, (const char*)u_h + r0 * es * p, (size_t)(r1 - r0) * es * p,
                                  cudaMemcpyHostToDevice, ctx->in)) || !ok(cudaEventRecord(wev[j], ctx->in)))
            return false;
        }
        timing_mark("chunk 0 input landed", ctx->in);
        return ok(cudaEventRecord(ev[0], ctx->in));
      }
      const bool r = ok(cudaMemcpyAsync((char*)h.u + b0[i] * in_row, (const char*)u_h + b0[i] * in_row,
                                        (size_t)(b0[i + 1] - b0[i]) * in_row, cudaMemcpyHostToDevice, ctx->in)) &&
                     ok(cudaEventRecord(ev[2 * i], ctx->in));
      timing_mark("chunk " + std::to_string(i) + " input landed", ctx->in);
      return r;
    };
    auto run_windows = [&](int i) {                   // one sequence: b0[i]
      const char* us = (const char*)h.u + b0[i] * in_row;
      char* ys = (char*)h.y + b0[i] * out_row;
      for (int j = 0; j < kW && rc == CASC_OK; ++j) {
        int64_t r0, r1;
        win(j, &r0, &r1);
        if (r1 <= r0) break;
        if (i == 0 && !ok(cudaStreamWaitEvent(st, wev[j], 0))) break;
        const int64_t a = std::max<int64_t>(0, r0 - Hu);
        rc = mimo_run(m, p, q, r1 - a, 1, Ne, N_max, mode, h.pack, D_h != nullptr, us + a * es * p, ys + r0 * es * q,
                      r0 - a, h.apply_ws, h.apply_bytes, st);
        if (rc) break;
        if (i == nc - 1) {                            // this window's output leaves now
          if (!ok(cudaEventRecord(wev[kW + j], st)) || !ok(cudaStreamWaitEvent(ctx->out, wev[kW + j], 0)) ||
              !ok(cudaMemcpyAsync((char*)y_h + b0[i] * out_row + r0 * es * q, ys + r0 * es * q,
                                  (size_t)(r1 - r0) * es * q, cudaMemcpyDeviceToHost, ctx->out)))
            break;
        }
      }
    };
    if (rc == CASC_OK && ok(cudaStreamWaitEvent(ctx->in, ctx->inputs_free, 0)) && submit(0)) {
      for (int i = 0; i < nc; ++i) {
        const bool wi = windowed(i);
        if (!(wi && i == 0) && !ok(cudaStreamWaitEvent(st, ev[2 * i], 0))) break;
        if (wi) {
          run_windows(i);
        } else {
          rc = mimo_run(m, p, q, L, b0[i + 1] - b0[i], Ne, N_max, mode, h.pack, D_h != nullptr,
                        (const char*)h.u + b0[i] * in_row, (char*)h.y + b0[i] * out_row, 0, h.apply_ws,
                        h.apply_bytes, st);
        }
        if (rc) break;
        timing_mark("chunk " + std::to_string(i) + " computed", st);
        if (!(wi && i == nc - 1)) {                   // the whole chunk's output
          if (!ok(cudaEventRecord(ev[2 * i + 1], st)) || !ok(cudaStreamWaitEvent(ctx->out, ev[2 * i + 1], 0)) ||
              !ok(cudaMemcpyAsync((char*)y_h + b0[i] * out_row, (const char*)h.y + b0[i] * out_row,
                                  (size_t)(b0[i + 1] - b0[i]) * out_row, cudaMemcpyDeviceToHost, ctx->out)))
            break;
        }
        if (i + 1 < nc && !submit(i + 1)) break;
      }
    }
    // drain all three streams before returning, also on error: no copy into or out of the caller's
    // host buffers may still be in flight, and the events are destroyed only once unused
    timing_mark("outputs copied", ctx->out);
    const cudaError_t e1 = cudaStreamSynchronize(ctx->out), e2 = cudaStreamSynchronize(st);
    const cudaError_t e3 = cudaStreamSynchronize(ctx->in);
    if (getenv("CASC_TIMING") && g_timing_t0) timing_print();
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (rc) return rc;
    return (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) ? CASC_ERR_CUDA : CASC_OK;
  }
  CASC_TRY(cudaMemcpyAsync(h.u, u_h, es * n_sys * batch * L * p, cudaMemcpyHostToDevice, st));
  rc = engine_powers(n_sys, m, N_host, N_max, h.Abar, mode, h.pack, st);
  if (rc) return rc;
  const int launches_powers = g_launches;
  rc = engine_apply(n_sys, m, p, q, L, batch, N_host, N_max, mode, h.pack, h.Bbar, h.C,
                    D_h ? h.D : nullptr, h.u, h.y, h.apply_ws, h.apply_bytes, st);
  if (rc) return rc;
  CASC_TRY(cudaMemcpyAsync(y_h, h.y, es * n_sys * batch * L * q, cudaMemcpyDeviceToHost, st));
  CASC_TRY(cudaStreamSynchronize(st));
  (void)launches_powers;
  return CASC_OK;
}

}  // extern "C"
