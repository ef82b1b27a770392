// Runtime plumbing of the C ABI: error TLS, launch counter, device queries.
#include <stdarg.h>
#include <stdio.h>

#include <atomic>

#include "wg_internal.cuh"

namespace {
thread_local char g_err[512] = "";
std::atomic<uint64_t> g_launches{0};
int g_sms = 0;
}  // namespace

namespace wg {

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int sm_count() {
  if (g_sms == 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      g_sms = n;
    else
      g_sms = 148;
  }
  return g_sms;
}

}  // namespace wg

extern "C" {

const char* wg_last_error(void) { return g_err; }

const char* wg_version(void) { return "wgb200 0.1.0 sm_100a"; }

uint64_t wg_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int wg_device_sms(int* sms) {
  int dev = 0;
  WG_CUDA_TRY(cudaGetDevice(&dev));
  WG_CUDA_TRY(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev));
  return WG_OK;
}

}  // extern "C"
