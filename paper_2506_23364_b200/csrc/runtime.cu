// Runtime plumbing of the C ABI: error TLS, launch counter, device queries.
#include <stdarg.h>
#include <stdio.h>

#include <atomic>
#include <mutex>

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

// Resident CTAs per SM of (kernel, block, dynamic smem), from the occupancy
// calculator, cached per (function, block, smem).
int resident_ctas(const void* fn, int block, size_t smem) {
  struct Entry {
    const void* fn;
    int block;
    size_t smem;
    int ctas;
  };
  static Entry cache[64];
  static std::atomic<int> used{0};
  static std::mutex mu;
  const int n = used.load(std::memory_order_acquire);
  for (int i = 0; i < n; i++)
    if (cache[i].fn == fn && cache[i].block == block && cache[i].smem == smem) return cache[i].ctas;
  int ctas = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, fn, block, smem) != cudaSuccess || ctas < 1) {
    cudaGetLastError();
    ctas = 1;
  }
  std::lock_guard<std::mutex> g(mu);
  const int k = used.load(std::memory_order_relaxed);
  if (k < 64) {
    cache[k] = Entry{fn, block, smem, ctas};
    used.store(k + 1, std::memory_order_release);
  }
  return ctas;
}

}  // namespace wg

namespace {
// Small device -> host readback written by the SMs straight into pinned
// (UVA-mapped) host memory: it does not queue behind bulk transfers on the
// device-to-host copy engine.
__global__ void peek_kernel(const unsigned long long* __restrict__ src, unsigned long long* dst, int n) {
  const int i = threadIdx.x;
  if (i < n) dst[i] = src[i];
}
}  // namespace

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

int wg_peek(const void* src, void* host_dst, int64_t nwords, void* stream) {
  if (nwords <= 0) return WG_OK;
  if (nwords > 1024) return wg::set_error(WG_EARG, "wg_peek reads at most 1024 words");
  if (!src || !host_dst) return wg::set_error(WG_EARG, "null buffer");
  if ((((uintptr_t)src) | ((uintptr_t)host_dst)) & 7) return wg::set_error(WG_EARG, "buffers must be 8-byte aligned");
  peek_kernel<<<1, 1024, 0, wg::as_stream(stream)>>>(reinterpret_cast<const unsigned long long*>(src),
                                                     reinterpret_cast<unsigned long long*>(host_dst), (int)nwords);
  WG_LAUNCH_CHECK("peek_kernel");
  return WG_OK;
}

}  // extern "C"
