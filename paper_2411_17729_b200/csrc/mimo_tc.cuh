// MIMO tensor-core path (bf16 storage): argument blocks and launchers (internal).
#pragma once
#include <cuda.h>
#include "common.cuh"

namespace casc {

struct MimoMaps {                 // passed as one __grid_constant__ kernel parameter
  CUtensorMap A[3];               // source signals [batch][L][K_src]   box {64, 128, 1}
  CUtensorMap W[3];               // weights [n_out][K_src]             box {64, BN}
  CUtensorMap R;                  // residual [batch][L][n_out]         box {64, 128, 1}
  CUtensorMap out;                // output   [batch][L][n_out]         box {64, 128, 1}
};
struct MimoArg {
  int n_src; int K[3]; int64_t shift[3];
  int64_t L; int batch; int n_out; int has_residual;
};
struct MimoSrc { const void* A; const void* W; int K; int64_t shift; };
struct MimoGemm {
  MimoSrc src[3]; int n_src;
  const void* R; void* out; int n_out;
  int64_t L; int batch;
};

bool mimo_tc_supported(int m, int p, int q);
// tf32 = true: 3xTF32 (fp32 signals, weights as [2][n_out][K] tf32 hi/lo); else bf16.
int launch_mimo_gemm(const MimoGemm& g, bool tf32, cudaStream_t st);

}  // namespace casc
