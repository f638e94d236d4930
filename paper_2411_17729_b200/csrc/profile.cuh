#pragma once
#include "common.cuh"

namespace casc {
enum KClass {
  K_POWERS = 0, K_PACK, K_DERIVED, K_FIRST, K_STAGE, K_LAST, K_DIRECT, K_CONVERT,
  K_BANK_HEAD, K_BANK_STAGE, K_BANK_TAIL, K_MIMO_STAGE, K_MIMO_FIRST, K_MIMO_LAST, K_SEQ_HALO, K_NCLASS
};
// math pipe of a launch's executed flops (the peak they are judged against)
enum KPipe { PIPE_NONE = 0, PIPE_TF32 = 1, PIPE_BF16 = 2, PIPE_FP64 = 3, PIPE_FP32 = 4 };

// RAII: records a start event now and an end event when it goes out of scope (after the
// launch it brackets), both on `st`, when profiling is enabled on this host thread.
class ProfScope {
 public:
  // bytes / flops: the ALGORITHMIC work of the launch (per-unit figure x units)
  ProfScope(cudaStream_t st, int cls, double bytes, double flops);
  ~ProfScope();
  // the EXECUTED work of the schedule run: HBM bytes the kernel must move and the math-pipe flops
  // it issues (3xTF32 = three tf32 products per source; zero blocks skipped are not executed)
  void exec(double bytes, double flops, int pipe);
  // A zeroed device counter (unsigned long long) the launch adds its ISSUED math-pipe flops to
  // (the kernel counts the MMAs it issues), or nullptr when profiling is off. When set, it replaces
  // the host estimate of exec() flops at read time.
  unsigned long long* device_flops();
  void drop_device_flops();            // the launch did not use the counter (host estimate stands)
 private:
  cudaStream_t st_;
  int idx_;
};
}  // namespace casc
