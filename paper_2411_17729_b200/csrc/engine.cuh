// Host engine entry points (internal).
#pragma once
#include <mutex>
#include <string>
#include "common.cuh"

namespace casc {
// Per-device host context of the host-buffer entry (casc_run_host) and the side streams of the
// engines: created once per device under a global lock, never freed (process lifetime).
//   mu      serialises casc_run_host calls on one device (they share the copy streams and the
//           pinned staging of the channel tables; the call is synchronous anyway)
//   in/out  copy-in / copy-out streams; side: the bank's pair-weight stream (apply paths)
struct DevCtx {
  std::mutex mu;
  cudaStream_t in = nullptr, out = nullptr, side = nullptr;
  cudaEvent_t inputs_free = nullptr;
  int* pinned = nullptr;
  size_t pinned_n = 0;
  int ensure_pinned(size_t n_ints);   // grow the pinned staging (caller holds mu)
  double* dnorm = nullptr;            // casc_powers_norms accumulators
  size_t dnorm_n = 0;
  int* dmeta = nullptr;               // device copy of the bank channel tables (all waves)
  size_t dmeta_n = 0;
  int ensure_dmeta(size_t n_ints);    // grow it (caller holds mu)
};
DevCtx* dev_ctx();                    // the current device's context; nullptr on a CUDA error
// CASC_TIMING diagnostics (bank_engine.cu): labelled events against the origin casc_run_host records
void timing_mark(const std::string& what, cudaStream_t s);
void timing_print();
extern cudaEvent_t g_timing_t0;

size_t apply_ws_bytes(int n, int m, int p, int q, int64_t L, int batch, int mode, int n_max);
// validate_common's result for a valid call with n, L or batch = 0 (the entry points return CASC_OK
// without touching any buffer)
constexpr int kEmptyCall = -1;
int validate_common(int n, int m, int p, int q, int64_t L, int batch, int N_max, int mode);
int engine_apply(int n, int m, int p, int q, int64_t L, int batch, const int* N_host, int N_max,
                 int mode, const void* pack, const double* Bbar, const double* C, const double* D,
                 const void* u, void* y, void* ws, size_t ws_bytes, cudaStream_t st);
bool bank_tc_path(int m, int p, int q, int mode);
size_t bank_ws_bytes(int n, int m, int64_t L, int batch, int n_max);
int engine_bank_tc(int n, int m, int64_t L, int batch, const int* N_host, int N_max, const void* pack,
                   const double* Bbar, const double* C, const double* D, const void* u, void* y, void* ws,
                   size_t ws_bytes, cudaStream_t st);
int engine_bank_pipelined(int n, int m, int64_t L, int batch, const int* N_host, int N_max, const void* pack,
                          const double* Bbar, const double* C, const double* D, float* u_dev, float* y_dev,
                          const void* u_h, const void* y_h, void* ws, size_t ws_bytes, cudaStream_t st,
                          DevCtx* ctx);
bool mimo_tc_path(int n, int m, int p, int q, int mode);
size_t mimo_ws_bytes(int m, int p, int q, int64_t L, int batch, int mode);
int engine_mimo_tc(int m, int p, int q, int64_t L, int batch, int N, int N_max, int mode, const void* pack,
                   const double* Bbar, const double* C, const double* D, const void* u, void* y, void* ws,
                   size_t ws_bytes, cudaStream_t st);
// MIMO workspace (mimo_engine.cu): derived float64 weights, their operand-format images, and the
// two state buffers of batch * L rows of m (ping-pong)
struct MimoWs {
  double *AB64, *CP64, *CBD64, *CAB64, *A2B64, *A3B64, *CP1_64, *CP3_64;
  void *Bb, *AB, *C, *CP, *D, *CBD, *CAB, *A2B, *A3B, *CP1, *CP3;   // operand-format weights (bf16, or tf32 hi/lo)
  void *Va, *Vb;
  size_t bytes;
};
MimoWs carve_mimo(void* ws, int m, int p, int q, int64_t L, int batch, int mode);
// derived weights of the fused first / last steps (R21): Abar Bbar, C P_Ne, C Bbar + D,
// C Abar Bbar, and for Ne >= 2 the Krylov head's Abar^2 Bbar, Abar^3 Bbar (R28), in float64 and
// rounded once to the GEMM operand format
int mimo_derive(int m, int p, int q, int Ne, const PackLayout& P, const double* Bbar, const double* C,
                const double* D, const MimoWs& w, bool tf32, cudaStream_t st);
// R31 (the MIMO output fold): with Ne >= 3 the last stage Ne-1 is folded into the output step,
// y = C v' + (C P_{Ne-1}) v'_{l-h} + (C P_Ne) v'_{l-2h} + (C P_Ne P_{Ne-1}) v'_{l-3h} + D u_l,
// v' = v^(Ne-1), h = 2^(Ne-1); the streaming stages run k0 .. Ne-2
inline bool mimo_fold(int Ne) { return Ne >= 3; }
// time rows of v the output step reads before l: 3 h (fold) or 2^Ne
inline int64_t mimo_out_halo(int Ne) { return Ne <= 0 ? 0 : (mimo_fold(Ne) ? 3 * ((int64_t)1 << (Ne - 1)) : (int64_t)1 << Ne); }
// the output step as a shifted GEMM over the buffer V holding v^(Ne) (or v^(Ne-1) with the fold):
// sources at row shifts (0, h, 2h, 3h) x unit (unit = batch for time-major shards, 1 otherwise),
// reading V and u with row0 halo rows in front; D (q x p) as the last source when present
struct MimoGemm;
void mimo_output_gemm(MimoGemm& g, const MimoWs& w, int Ne, int m, int p, int q, const void* V, int64_t v_row0,
                      const void* u, int64_t u_row0, bool has_D, int64_t unit);
// the MIMO cascade steps with the derived weights already in ws (engine_mimo_tc = derive + run);
// out_skip: leading window rows of history that are not written to y (batch == 1)
int mimo_run(int m, int p, int q, int64_t L, int batch, int Ne, int N_max, int mode, const void* pack, bool has_D,
             const void* u, void* y, int64_t out_skip, void* ws, size_t ws_bytes, cudaStream_t st);
int engine_powers(int n, int m, const int* N_host, int N_max, const double* Abar, int mode,
                  void* pack, cudaStream_t st);
}  // namespace casc
