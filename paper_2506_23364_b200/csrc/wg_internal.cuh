// Internal helpers shared by the wgb200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/wgb200.h"

namespace wg {

// thread-local error message + launch counter (runtime.cu)
int set_error(int code, const char* fmt, ...);
void count_launch();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();

// Grid size for a streaming (HBM-bound) kernel: enough resident CTAs to cover
// every SM several times, never more blocks than work.
inline int stream_grid(int64_t work_items, int block, int ctas_per_sm = 8) {
  int64_t want = (work_items + block - 1) / block;
  int64_t cap = (int64_t)sm_count() * ctas_per_sm;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return (int)want;
}

}  // namespace wg

#define WG_LAUNCH_CHECK(what)                                                        \
  do {                                                                               \
    cudaError_t _e = cudaGetLastError();                                             \
    if (_e != cudaSuccess) return wg::set_error(WG_ECUDA, "%s: %s", what, cudaGetErrorString(_e)); \
    wg::count_launch();                                                              \
  } while (0)

#define WG_CUDA_TRY(call)                                                            \
  do {                                                                               \
    cudaError_t _e = (call);                                                         \
    if (_e != cudaSuccess) return wg::set_error(WG_ECUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
  } while (0)
