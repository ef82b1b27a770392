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

// Grid for a grid-stride kernel: exactly the CTAs that are resident at once
// (occupancy calculator: registers, shared memory, block size), never more
// than the work needs -- one balanced wave, no tail wave of leftover blocks.
int resident_ctas(const void* fn, int block, size_t smem);

template <typename Kernel>
inline int resident_grid(Kernel* kernel, int64_t work_items, int block, size_t smem = 0) {
  int64_t want = (work_items + block - 1) / block;
  const int64_t cap = (int64_t)sm_count() * resident_ctas(reinterpret_cast<const void*>(kernel), block, smem);
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
