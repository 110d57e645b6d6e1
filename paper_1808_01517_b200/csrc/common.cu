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
// kernel timer (dl_ktimer_*): per slot a ring of (begin, end) event pairs, one pair per bracketed launch
constexpr int kKtRing = 64;
bool g_kt_armed = false;
cudaEvent_t g_kt_ev[2][kKtRing][2] = {};
int64_t g_kt_n[2] = {0, 0};   // launches bracketed per slot (the ring holds the last kKtRing)
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

int ktimer_record(int slot, int end, cudaStream_t st) {
  if (!g_kt_armed || slot < 0 || slot > 1) return DL_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  DL_CUDA(cudaStreamIsCapturing(st, &cs));
  cudaEvent_t ev = g_kt_ev[slot][g_kt_n[slot] % kKtRing][end];
  if (cs == cudaStreamCaptureStatusActive)   // an external event node: every graph replay re-records it
    DL_CUDA(cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal));
  else
    DL_CUDA(cudaEventRecord(ev, st));
  if (end) ++g_kt_n[slot];
  return DL_OK;
}

}  // namespace dl

extern "C" {

int dl_ktimer_arm(int on) {
  if (on && !g_kt_ev[0][0][0])
    for (auto& ring : g_kt_ev)
      for (auto& pair : ring)
        for (auto& ev : pair) DL_CUDA(cudaEventCreate(&ev));
  g_kt_armed = on != 0;
  return DL_OK;
}

int64_t dl_ktimer_count(int slot) { return slot == 0 || slot == 1 ? g_kt_n[slot] : -1; }

int dl_ktimer_read(int slot, int back, float* ms) {
  DL_REQUIRE(slot == 0 || slot == 1, "ktimer_read: slot %d (0 forward, 1 adjoint)", slot);
  DL_REQUIRE(ms && g_kt_ev[0][0][0], "ktimer_read: timer never armed or null output");
  DL_REQUIRE(back >= 0 && back < kKtRing && back < g_kt_n[slot],
             "ktimer_read: launch %d back of %lld bracketed (ring of %d)", back, (long long)g_kt_n[slot], kKtRing);
  const auto& pair = g_kt_ev[slot][(g_kt_n[slot] - 1 - back) % kKtRing];
  DL_CUDA(cudaEventElapsedTime(ms, pair[0], pair[1]));
  return DL_OK;
}

int dl_abi_version(void) { return 104; }

const char* dl_last_error(void) { return g_err; }

int dl_last_launch_count(void) { return g_launches; }

int64_t dl_total_launch_count(void) { return g_total_launches.load(std::memory_order_relaxed); }

int dl_device_supported(void) { return dl::device_check(nullptr) == DL_OK ? 1 : 0; }

}  // extern "C"
