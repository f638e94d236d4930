// Host engine entry points (internal).
#pragma once
#include <mutex>
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
};
DevCtx* dev_ctx();                    // the current device's context; nullptr on a CUDA error

size_t apply_ws_bytes(int n, int m, int p, int q, int64_t L, int batch, int mode, int n_max);
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
  double *AB64, *CP64, *CBD64, *CAB64, *A2B64, *A3B64;
  void *Bb, *AB, *C, *CP, *D, *CBD, *CAB, *A2B, *A3B;   // operand-format weights (bf16, or tf32 hi/lo planes)
  void *Va, *Vb;
  size_t bytes;
};
MimoWs carve_mimo(void* ws, int m, int p, int q, int64_t L, int batch, int mode);
// derived weights of the fused first / last steps (R21): Abar Bbar, C P_Ne, C Bbar + D,
// C Abar Bbar, and for Ne >= 2 the Krylov head's Abar^2 Bbar, Abar^3 Bbar (R28), in float64 and
// rounded once to the GEMM operand format
int mimo_derive(int m, int p, int q, int Ne, const PackLayout& P, const double* Bbar, const double* C,
                const double* D, const MimoWs& w, bool tf32, cudaStream_t st);
// the MIMO cascade steps with the derived weights already in ws (engine_mimo_tc = derive + run);
// out_skip: leading window rows of history that are not written to y (batch == 1)
int mimo_run(int m, int p, int q, int64_t L, int batch, int Ne, int N_max, int mode, const void* pack, bool has_D,
             const void* u, void* y, int64_t out_skip, void* ws, size_t ws_bytes, cudaStream_t st);
int engine_powers(int n, int m, const int* N_host, int N_max, const double* Abar, int mode,
                  void* pack, cudaStream_t st);
}  // namespace casc
