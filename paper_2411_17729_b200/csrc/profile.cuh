#pragma once
#include "common.cuh"

namespace casc {
enum KClass {
  K_POWERS = 0, K_PACK, K_DERIVED, K_FIRST, K_STAGE, K_LAST, K_DIRECT, K_CONVERT,
  K_BANK_HEAD, K_BANK_STAGE, K_BANK_TAIL, K_MIMO_STAGE, K_MIMO_FIRST, K_MIMO_LAST, K_BANK_FUSED, K_NCLASS
};

// RAII: records a start event now and an end event when it goes out of scope (after the
// launch it brackets), both on `st`, when profiling is enabled on this host thread.
class ProfScope {
 public:
  ProfScope(cudaStream_t st, int cls, double bytes, double flops);
  ~ProfScope();
 private:
  cudaStream_t st_;
  int idx_;
};
}  // namespace casc
