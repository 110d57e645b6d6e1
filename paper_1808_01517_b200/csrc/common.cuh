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

// Kernel timer: when armed (dl_ktimer_arm), record slot's begin (end = 0) or end event on st.
int ktimer_record(int slot, int end, cudaStream_t st);

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
