// Optional per-kernel-class timing: when enabled on the calling host thread, each launch of
// the engine is bracketed by CUDA events recorded on the launch stream, and tagged with the
// algorithmic bytes / flops of that launch. bench.py reads these to report the dominant
// kernel's achieved bandwidth or throughput (roofline) from live, in-run measurements.
#include <vector>
#include "common.cuh"
#include "profile.cuh"

namespace casc {

struct ProfRec {
  cudaEvent_t a, b;
  int cls;
  double bytes, flops;
  double xbytes, xflops;   // executed (ProfScope::exec); default = algorithmic
  int pipe;
  int counter;             // index of a device flop counter (device_flops), -1: none
};
struct ProfState {
  bool on = false;
  std::vector<ProfRec> recs;
  unsigned long long* counters = nullptr;   // device [kCounters]
  int n_counters = 0;
  static constexpr int kCounters = 1 << 16;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};
static thread_local ProfState g_prof;

ProfScope::ProfScope(cudaStream_t st, int cls, double bytes, double flops) : st_(st), idx_(-1) {
  if (!g_prof.on) return;
  ProfRec r{g_prof.get(), g_prof.get(), cls, bytes, flops, bytes, flops, PIPE_NONE, -1};
  cudaEventRecord(r.a, st);
  g_prof.recs.push_back(r);
  idx_ = (int)g_prof.recs.size() - 1;
}
void ProfScope::exec(double bytes, double flops, int pipe) {
  if (idx_ < 0) return;
  ProfRec& r = g_prof.recs[idx_];
  r.xbytes = bytes;
  r.xflops = flops;
  r.pipe = pipe;
}
// the counters are allocated and zeroed by casc_profile_enable / casc_profile_reset (outside any
// timed region): a scope only takes the next slot
unsigned long long* ProfScope::device_flops() {
  if (idx_ < 0 || !g_prof.counters || g_prof.n_counters >= ProfState::kCounters) return nullptr;
  const int i = g_prof.n_counters++;
  g_prof.recs[idx_].counter = i;
  return g_prof.counters + i;
}
void ProfScope::drop_device_flops() {
  if (idx_ >= 0) g_prof.recs[idx_].counter = -1;
}
ProfScope::~ProfScope() {
  if (idx_ >= 0) cudaEventRecord(g_prof.recs[idx_].b, st_);
}

static const char* kNames[K_NCLASS] = {"powers_square", "powers_pack", "derived", "first_stage",
                                       "stage", "last_stage", "direct", "convert",
                                       "bank_head", "bank_stage", "bank_tail", "mimo_tc_stage",
                                       "mimo_tc_first", "mimo_tc_last", "seq_halo"};

}  // namespace casc

using namespace casc;
extern "C" {

static int zero_counters() {
  if (!g_prof.counters &&
      cudaMalloc(&g_prof.counters, sizeof(unsigned long long) * ProfState::kCounters) != cudaSuccess) {
    g_prof.counters = nullptr;
    return CASC_ERR_CUDA;
  }
  if (cudaMemset(g_prof.counters, 0, sizeof(unsigned long long) * ProfState::kCounters) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess)
    return CASC_ERR_CUDA;
  g_prof.n_counters = 0;
  return CASC_OK;
}

// Diagnostics mode (bench.py): enabling allocates and zeroes the device counters once, synchronously.
int casc_profile_enable(int on) {
  g_prof.on = on != 0;
  if (g_prof.on && g_prof.n_counters == 0 && !g_prof.counters) return zero_counters();
  return CASC_OK;
}

int casc_profile_reset(void) {
  for (auto& r : g_prof.recs) {
    g_prof.pool.push_back(r.a);
    g_prof.pool.push_back(r.b);
  }
  g_prof.recs.clear();
  if (g_prof.counters) return zero_counters();
  g_prof.n_counters = 0;
  return CASC_OK;
}

int casc_profile_num_classes(void) { return K_NCLASS; }

const char* casc_profile_class_name(int cls) {
  return (cls >= 0 && cls < K_NCLASS) ? kNames[cls] : "unknown";
}

int casc_profile_read(int cls, int* launches, double* ms, double* bytes, double* flops) {
  int n = 0;
  double t = 0, by = 0, fl = 0;
  for (auto& r : g_prof.recs) {
    if (r.cls != cls) continue;
    if (cudaEventSynchronize(r.b) != cudaSuccess) return CASC_ERR_CUDA;
    float e = 0.f;
    if (cudaEventElapsedTime(&e, r.a, r.b) != cudaSuccess) return CASC_ERR_CUDA;
    ++n;
    t += e;
    by += r.bytes;
    fl += r.flops;
  }
  if (launches) *launches = n;
  if (ms) *ms = t;
  if (bytes) *bytes = by;
  if (flops) *flops = fl;
  return CASC_OK;
}

int casc_profile_read_exec(int cls, double* exec_bytes, double* exec_flops, int* pipe) {
  double by = 0, fl = 0;
  int pp = PIPE_NONE;
  for (auto& r : g_prof.recs) {
    if (r.cls != cls) continue;
    by += r.xbytes;
    if (r.counter >= 0) {                   // counted by the kernel itself
      unsigned long long v = 0;
      if (cudaEventSynchronize(r.b) != cudaSuccess ||
          cudaMemcpy(&v, g_prof.counters + r.counter, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess)
        return CASC_ERR_CUDA;
      fl += (double)v;
    } else {
      fl += r.xflops;
    }
    if (r.pipe != PIPE_NONE) pp = r.pipe;
  }
  if (exec_bytes) *exec_bytes = by;
  if (exec_flops) *exec_flops = fl;
  if (pipe) *pipe = pp;
  return CASC_OK;
}

}  // extern "C"
