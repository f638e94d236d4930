// Host sequencing of the MIMO tensor-core path (one system, bf16 storage; m, p, q multiples
// of 64). Same step schedule as the generic engine (cascade_api.cu), each step one launch of
// the shifted multi-source tcgen05 GEMM (mimo_tc.cu):
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

__global__ void f64_to_bf16_kernel(const double* src, __nv_bfloat16* dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn((float)src[i]);
}
int launch_f64_to_bf16(const double* src, __nv_bfloat16* dst, int64_t n, cudaStream_t st) {
  if (n <= 0) return CASC_OK;
  f64_to_bf16_kernel<<<(int)std::min<int64_t>(ceil_div(n, 256), 148 * 8), 256, 0, st>>>(src, dst, n);
  CASC_LAUNCHED();
  return CASC_OK;
}

struct MimoWs {
  double *AB64, *CP64, *CBD64, *CAB64;
  __nv_bfloat16 *Bb, *AB, *C, *CP, *D, *CBD, *CAB;
  void *Va, *Vb;
  size_t bytes;
};

static MimoWs carve_mimo(void* ws, int m, int p, int q, int64_t L, int batch) {
  Carver c(ws);
  MimoWs w{};
  w.AB64 = c.take<double>((size_t)m * p);
  w.CP64 = c.take<double>((size_t)q * m);
  w.CBD64 = c.take<double>((size_t)q * p);
  w.CAB64 = c.take<double>((size_t)q * p);
  w.Bb = c.take<__nv_bfloat16>((size_t)m * p);
  w.AB = c.take<__nv_bfloat16>((size_t)m * p);
  w.C = c.take<__nv_bfloat16>((size_t)q * m);
  w.CP = c.take<__nv_bfloat16>((size_t)q * m);
  w.D = c.take<__nv_bfloat16>((size_t)q * p);
  w.CBD = c.take<__nv_bfloat16>((size_t)q * p);
  w.CAB = c.take<__nv_bfloat16>((size_t)q * p);
  const size_t vbytes = (size_t)batch * (size_t)L * m * 2;
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
  return !force_simt && n == 1 && mode == CASC_BF16 && mimo_tc_supported(m, p, q);
}

size_t mimo_ws_bytes(int m, int p, int q, int64_t L, int batch) { return carve_mimo(nullptr, m, p, q, L, batch).bytes; }

static int eff_order_m(int N, int64_t L) {
  if (L <= 2) return 0;
  int kstar = 0;
  while (((int64_t)1 << (kstar + 1)) < L) ++kstar;
  return N < kstar ? N : kstar;
}

int engine_mimo_tc(int m, int p, int q, int64_t L, int batch, int N, int N_max, const void* pack,
                   const double* Bbar, const double* C, const double* D, const void* u, void* y, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  MimoWs w = carve_mimo(ws, m, p, q, L, batch);
  if (ws_bytes < w.bytes) return CASC_ERR_WORKSPACE;
  PackLayout P = pack_layout(const_cast<void*>(pack), 1, m, N_max, CASC_BF16);
  const int64_t mm = (int64_t)m * m;
  const int Ne = eff_order_m(N, L);
  int rc;
  {
    ProfScope ps(st, K_DERIVED, 0.0, 2.0 * ((double)m * m * p + (double)q * m * m + 2.0 * q * m * p));
    DgemmArg a{};
    a.M = m; a.N = p; a.K = m;                                     // Abar Bbar
    a.A = P.p64; a.lda = m; a.B = Bbar; a.ldb = p; a.C = w.AB64; a.ldc = p;
    if ((rc = launch_dgemm(a, 1, st))) return rc;
    a = DgemmArg{};                                                // C P_Ne
    a.M = q; a.N = m; a.K = m;
    a.A = C; a.lda = m; a.B = P.p64 + Ne * mm; a.ldb = m; a.C = w.CP64; a.ldc = m;
    if ((rc = launch_dgemm(a, 1, st))) return rc;
    a = DgemmArg{};                                                // C Bbar + D
    a.M = q; a.N = p; a.K = m;
    a.A = C; a.lda = m; a.B = Bbar; a.ldb = p; a.C = w.CBD64; a.ldc = p; a.Cadd = D;
    if ((rc = launch_dgemm(a, 1, st))) return rc;
    a = DgemmArg{};                                                // C Abar Bbar
    a.M = q; a.N = p; a.K = m;
    a.A = C; a.lda = m; a.B = w.AB64; a.ldb = p; a.C = w.CAB64; a.ldc = p;
    if ((rc = launch_dgemm(a, 1, st))) return rc;
    if ((rc = launch_f64_to_bf16(Bbar, w.Bb, (int64_t)m * p, st))) return rc;
    if ((rc = launch_f64_to_bf16(w.AB64, w.AB, (int64_t)m * p, st))) return rc;
    if ((rc = launch_f64_to_bf16(C, w.C, (int64_t)q * m, st))) return rc;
    if ((rc = launch_f64_to_bf16(w.CP64, w.CP, (int64_t)q * m, st))) return rc;
    if ((rc = launch_f64_to_bf16(w.CBD64, w.CBD, (int64_t)q * p, st))) return rc;
    if ((rc = launch_f64_to_bf16(w.CAB64, w.CAB, (int64_t)q * p, st))) return rc;
    if (D && (rc = launch_f64_to_bf16(D, w.D, (int64_t)q * p, st))) return rc;
  }
  const double rows = (double)batch * L;
  if (Ne == 0) {
    MimoGemm g{};
    g.src[0] = {u, w.CBD, p, 0};
    g.src[1] = {u, w.CAB, p, 1};
    g.n_src = 2; g.out = y; g.n_out = q; g.L = L; g.batch = batch;
    ProfScope ps(st, K_MIMO_LAST, rows * (p + q) * 2.0, rows * 4.0 * q * p);
    return launch_mimo_gemm_bf16(g, st);
  }
  {
    MimoGemm g{};
    g.src[0] = {u, w.Bb, p, 0};
    g.src[1] = {u, w.AB, p, 1};
    g.n_src = 2; g.out = w.Va; g.n_out = m; g.L = L; g.batch = batch;
    ProfScope ps(st, K_MIMO_FIRST, rows * (p + m) * 2.0, rows * 4.0 * m * p);
    if ((rc = launch_mimo_gemm_bf16(g, st))) return rc;
  }
  for (int k = 1; k <= Ne - 1; ++k) {
    void* Vs = (k - 1) % 2 == 0 ? w.Va : w.Vb;
    void* Vd = (k % 2 == 0) ? w.Va : w.Vb;
    MimoGemm g{};
    g.src[0] = {Vs, P.b16 + k * mm, m, (int64_t)1 << k};
    g.n_src = 1; g.R = Vs; g.out = Vd; g.n_out = m; g.L = L; g.batch = batch;
    ProfScope ps(st, K_MIMO_STAGE, rows * m * 2.0 * 2.0, rows * 2.0 * (double)mm);
    if ((rc = launch_mimo_gemm_bf16(g, st))) return rc;
  }
  {
    void* V = (Ne - 1) % 2 == 0 ? w.Va : w.Vb;
    MimoGemm g{};
    g.src[0] = {V, w.C, m, 0};
    g.src[1] = {V, w.CP, m, (int64_t)1 << Ne};
    g.n_src = 2;
    if (D) { g.src[2] = {u, w.D, p, 0}; g.n_src = 3; }
    g.out = y; g.n_out = q; g.L = L; g.batch = batch;
    ProfScope ps(st, K_MIMO_LAST, rows * (m + p + q) * 2.0, rows * (4.0 * q * m + 2.0 * q * p));
    if ((rc = launch_mimo_gemm_bf16(g, st))) return rc;
  }
  return CASC_OK;
}

}  // namespace casc
