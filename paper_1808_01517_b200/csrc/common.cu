// Status, error strings and device checks for the C ABI.
#include <stdarg.h>
#include <stdio.h>

#include <atomic>

#include "common.cuh"

namespace {
thread_local char g_err[512] = "";
thread_local int g_launches = 0;
std::atomic<int64_t> g_total_launches{0};
int g_sm_count[64] = {0};   // per device ordinal, 0 = unknown
int g_supported[64] = {0};  // 1 ok, -1 unsupported, 0 unknown
// kernel timer (dl_ktimer_*): one device trace buffer per device ordinal, allocated on the first arm
bool g_kt_armed = false;
dl::KTrace* g_kt_buf[64] = {};
}  // namespace

namespace dl {

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

void begin_call() { g_launches = 0; }

int after_launch(const char* what) {
  ++g_launches;
  g_total_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(DL_ECUDA, "launch of %s failed: %s", what, cudaGetErrorString(e));
  }
  return DL_OK;
}

int device_check(int* sm_count) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(DL_ENODEVICE, "no CUDA device: %s", cudaGetErrorString(e));
  }
  if (dev < 0 || dev >= 64) return fail(DL_ENODEVICE, "device ordinal %d out of range", dev);
  if (g_supported[dev] == 0) {
    cudaDeviceProp p;
    e = cudaGetDeviceProperties(&p, dev);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(DL_ENODEVICE, "cudaGetDeviceProperties: %s", cudaGetErrorString(e));
    }
    g_supported[dev] = (p.major == 10 && p.minor == 0) ? 1 : -1;
    g_sm_count[dev] = p.multiProcessorCount;
    if (g_supported[dev] < 0)
      return fail(DL_ENODEVICE, "device %d is sm_%d%d; this library is built for sm_100a only", dev,
                  p.major, p.minor);
  }
  if (g_supported[dev] < 0) return fail(DL_ENODEVICE, "device %d is not sm_100", dev);
  if (sm_count) *sm_count = g_sm_count[dev];
  return DL_OK;
}

KTrace* ktrace() {
  if (!g_kt_armed) return nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return nullptr;
  }
  return g_kt_buf[dev];
}

}  // namespace dl

extern "C" {

int dl_ktimer_arm(int on) {
  if (on) {
    int dev = 0;
    DL_CUDA(cudaGetDevice(&dev));
    DL_REQUIRE(dev >= 0 && dev < 64, "ktimer_arm: device ordinal %d out of range", dev);
    if (!g_kt_buf[dev]) {
      dl::KTrace h{};
      for (int s = 0; s < dl::kKtSlots; ++s) h.t[s][0][0] = ~0ull;
      DL_CUDA(cudaMalloc(&g_kt_buf[dev], sizeof(dl::KTrace)));
      DL_CUDA(cudaMemcpy(g_kt_buf[dev], &h, sizeof h, cudaMemcpyHostToDevice));
    }
  }
  g_kt_armed = on != 0;
  return DL_OK;
}

namespace {
int ktimer_snapshot(dl::KTrace* h) {
  int dev = 0;
  DL_CUDA(cudaGetDevice(&dev));
  DL_REQUIRE(dev >= 0 && dev < 64 && g_kt_buf[dev], "ktimer: never armed on device %d", dev);
  DL_CUDA(cudaDeviceSynchronize());
  DL_CUDA(cudaMemcpy(h, g_kt_buf[dev], sizeof *h, cudaMemcpyDeviceToHost));
  return DL_OK;
}
}  // namespace

int64_t dl_ktimer_count(int slot) {
  if (slot < 0 || slot >= dl::kKtSlots) return -1;
  dl::KTrace h;
  if (ktimer_snapshot(&h) != DL_OK) return -1;
  return (int64_t)h.seq[slot];
}

int dl_ktimer_read(int slot, int back, float* ms) {
  DL_REQUIRE(slot >= 0 && slot < dl::kKtSlots, "ktimer_read: slot %d (0 forward, 1 adjoint, 2 Gram)", slot);
  DL_REQUIRE(ms, "ktimer_read: null output");
  dl::KTrace h;
  DL_TRY(ktimer_snapshot(&h));
  const int64_t n = (int64_t)h.seq[slot];
  DL_REQUIRE(back >= 0 && back < dl::kKtRing - 1 && back < n,
             "ktimer_read: launch %d back of %lld recorded (ring of %d)", back, (long long)n, dl::kKtRing);
  const auto& e = h.t[slot][(n - 1 - back) % dl::kKtRing];
  DL_REQUIRE(e[1] >= e[0] && e[0] != ~0ull, "ktimer_read: incomplete record");
  *ms = (float)((double)(e[1] - e[0]) * 1e-6);
  return DL_OK;
}

int dl_abi_version(void) { return 105; }

const char* dl_last_error(void) { return g_err; }

int dl_last_launch_count(void) { return g_launches; }

int64_t dl_total_launch_count(void) { return g_total_launches.load(std::memory_order_relaxed); }

int dl_device_supported(void) { return dl::device_check(nullptr) == DL_OK ? 1 : 0; }

}  // extern "C"
