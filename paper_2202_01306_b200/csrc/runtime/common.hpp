// common.hpp -- error reporting and launch accounting shared by kernels and runtime.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "../../../include/harmony_b200.h"

namespace hm {

void set_last_error(const std::string &msg);

inline int fail(int code, const std::string &msg) {
  set_last_error(msg);
  return code;
}

// Kernels launched by this library (all threads); the bench reports the
// delta over its timed region as "gpu_launches".
std::atomic<int64_t> &launch_counter();
inline void count_launch(int64_t n = 1) { launch_counter().fetch_add(n, std::memory_order_relaxed); }
// SMs of the calling thread's current device (persistent kernels size their grid with it)
inline int current_sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      n <= 0)
    n = 148;
  return n;
}

// Optional per-launch timing hook (set by the runtime while profiling).
enum KernelClass { KC_GEMM = 0, KC_ATTN_FWD, KC_ATTN_BWD, KC_LAYERNORM, KC_XENT, KC_ADAM, KC_MISC, KC_COUNT };
struct KernelProfiler {
  virtual void begin(int cls, cudaStream_t s) = 0;
  virtual void end(int cls, cudaStream_t s, double flops, double bytes) = 0;
  // device {~first CTA start, last CTA end} globaltimer pair for the launch just
  // begun (atomicMax targets, zeroed before the profiled iteration), or null
  virtual unsigned long long *span_slot() { return nullptr; }
  virtual ~KernelProfiler() = default;
};
KernelProfiler *&profiler();
struct ProfScope {
  int cls;
  cudaStream_t s;
  double flops, bytes;
  ProfScope(int c, cudaStream_t st, double f, double b) : cls(c), s(st), flops(f), bytes(b) {
    if (profiler()) profiler()->begin(cls, s);
  }
  ~ProfScope() {
    if (profiler()) profiler()->end(cls, s, flops, bytes);
  }
};

#define HM_CUDA(call)                                                                        \
  do {                                                                                       \
    cudaError_t _e = (call);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return ::hm::fail(HM_ERR_DEVICE, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define HM_TRY(expr)         \
  do {                       \
    int _rc = (expr);        \
    if (_rc != HM_OK) return _rc; \
  } while (0)

}  // namespace hm
