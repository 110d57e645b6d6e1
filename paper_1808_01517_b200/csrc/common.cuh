// Shared helpers for libdelimit_sm100a.so: status handling, launch accounting,
// device queries.  All kernels are compiled for sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/delimit.h"

namespace dl {

// Record a message for dl_last_error() and return `code`.
int fail(int code, const char* fmt, ...);
// Check cudaPeekAtLastError after a launch; counts the launch.
int after_launch(const char* what);
// Reset the per-call launch counter (each public entry calls this first).
void begin_call();
// Validate the current device is sm_100 and return its SM count (cached per device).
int device_check(int* sm_count);

// Kernel timer (dl_ktimer_*): device-side launch timestamps.  Armed kernels take a KTrace pointer and stamp
// %globaltimer when their first CTA starts (min over CTAs) and their last CTA ends (max over CTAs) into a
// per-slot ring; the last CTA to finish advances the ring.  Works the same eagerly and inside replayed CUDA
// graphs (the pointer is a kernel argument, so every replay records), and measures the kernel alone.
constexpr int kKtSlots = 4;   // 0 forward chain, 1 adjoint chain, 2 Gram, 3 reserved
constexpr int kKtRing = 64;
struct KTrace {
  unsigned long long seq[kKtSlots];
  unsigned int done[kKtSlots];
  unsigned long long t[kKtSlots][kKtRing][2];
};
// The current device's trace buffer when the timer is armed, else null.
KTrace* ktrace();

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// thread 0 of every CTA, first thing in the kernel
__device__ __forceinline__ void ktrace_begin(KTrace* kt, int slot) {
  if (kt && threadIdx.x == 0) {
    const unsigned long long s = *(volatile unsigned long long*)&kt->seq[slot];
    atomicMin(&kt->t[slot][s % kKtRing][0], globaltimer_ns());
  }
}
// thread 0 of every CTA, after the CTA's last barrier
__device__ __forceinline__ void ktrace_end(KTrace* kt, int slot) {
  if (kt && threadIdx.x == 0) {
    const unsigned long long s = *(volatile unsigned long long*)&kt->seq[slot];
    atomicMax(&kt->t[slot][s % kKtRing][1], globaltimer_ns());
    __threadfence();
    if (atomicAdd(&kt->done[slot], 1u) == gridDim.x - 1) {   // last CTA: open the next ring entry
      __threadfence();
      const unsigned long long n = (s + 1) % kKtRing;
      kt->t[slot][n][0] = ~0ull;
      kt->t[slot][n][1] = 0ull;
      kt->done[slot] = 0u;
      __threadfence();
      *(volatile unsigned long long*)&kt->seq[slot] = s + 1;
    }
  }
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

template <typename T>
__host__ __device__ __forceinline__ T ceil_div(T a, T b) { return (a + b - 1) / b; }

}  // namespace dl

#define DL_REQUIRE(cond, ...)                                    \
  do {                                                           \
    if (!(cond)) return ::dl::fail(DL_EINVAL, __VA_ARGS__);      \
  } while (0)

#define DL_CUDA(call)                                                               \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return ::dl::fail(DL_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_));  \
  } while (0)

#define DL_TRY(expr)             \
  do {                           \
    int st_ = (expr);            \
    if (st_ != DL_OK) return st_; \
  } while (0)
