// L2 access-rate probe for the trajectory kernel's memory pattern (its DRAM
// traffic is ~1 % of the algorithmic bytes: the DEM patch gathers and the
// raster atomics are served by the 126 MB L2).  Working set: 96 MiB, inside
// L2.  Every thread walks its own SplitMix64 stream of random slots; all SMs,
// 32 warps per SM (the trajectory kernel's residency).  Prints one JSON line
// per probe:
//   gather32 : one 32-byte load (ld.global.nc.v4.f64) per op  -- the patch gather
//   red_add  : one 8-byte RED.ADD.64 per op                   -- the visit count
//   red_max  : one 8-byte RED.MAX.64 per op                   -- the drop max
//   step     : gather32 + red_add + red_max per op, the three to the same
//              kind of slots the trajectory step touches (a memory-only step)
//   *_red    : the same with the reductions issued as PTX red (REDG) instead
//              of atomicAdd / atomicMax with an unused result (ATOMG to RZ) --
//              what the trajectory kernel uses
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_peak l2_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

template <int kMode>
__global__ void __launch_bounds__(128, 8) probe(const double* __restrict__ quad, unsigned long long* hits,
                                                unsigned long long* zmax, unsigned long long nslots, int iters,
                                                double* sink) {
  unsigned long long s = mix(blockIdx.x * 128ull + threadIdx.x + 1);
  double acc = 0.0;
  for (int i = 0; i < iters; i++) {
    s += 0x9E3779B97F4A7C15ULL;
    const unsigned long long h = mix(s);
    const unsigned long long slot = (unsigned long long)(((unsigned __int128)h * nslots) >> 64);
    if (kMode == 0 || kMode == 3) {
      double a, b, c, d;
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(quad + 4 * slot));
      acc += a + b + c + d;
    }
    if (kMode == 1 || kMode == 3) atomicAdd(hits + slot, 1ULL);
    if (kMode == 2 || kMode == 3) atomicMax(zmax + slot, h >> 12);
    if (kMode == 4 || kMode == 6) asm volatile("red.global.add.u64 [%0], 1;" ::"l"(hits + slot) : "memory");
    if (kMode == 5 || kMode == 6) asm volatile("red.global.max.u64 [%0], %1;" ::"l"(zmax + slot), "l"(h >> 12) : "memory");
    if (kMode == 6) {
      double a, b, c, d;
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(quad + 4 * slot));
      acc += a + b + c + d;
    }
  }
  if (acc == 1.2345) sink[0] = acc;
}

int main() {
  const size_t quad_bytes = 64ull << 20, raster_bytes = 16ull << 20;  // 64 + 2 x 16 MiB = 96 MiB
  const unsigned long long nslots = raster_bytes / 8;                 // quad: 32 B per slot
  double* quad;
  unsigned long long *hits, *zmax;
  double* sink;
  cudaMalloc(&quad, quad_bytes);
  cudaMalloc(&hits, raster_bytes);
  cudaMalloc(&zmax, raster_bytes);
  cudaMalloc(&sink, 8);
  cudaMemset(quad, 0, quad_bytes);
  cudaMemset(hits, 0, raster_bytes);
  cudaMemset(zmax, 0, raster_bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, iters = 4096;
  const double ops = (double)blocks * 128 * iters;
  const char* names[7] = {"gather32", "red_add", "red_max", "step", "red_add_red", "red_max_red", "step_red"};
  for (int mode = 0; mode < 7; mode++) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
      cudaEventRecord(e0);
      switch (mode) {
        case 0: probe<0><<<blocks, 128>>>(quad, hits, zmax, nslots, iters, sink); break;
        case 1: probe<1><<<blocks, 128>>>(quad, hits, zmax, nslots, iters, sink); break;
        case 2: probe<2><<<blocks, 128>>>(quad, hits, zmax, nslots, iters, sink); break;
        case 3: probe<3><<<blocks, 128>>>(quad, hits, zmax, nslots, iters, sink); break;
        case 4: probe<4><<<blocks, 128>>>(quad, hits, zmax, nslots, iters, sink); break;
        case 5: probe<5><<<blocks, 128>>>(quad, hits, zmax, nslots, iters, sink); break;
        default: probe<6><<<blocks, 128>>>(quad, hits, zmax, nslots, iters, sink); break;
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;  // rep 0 warms L2
    }
    const double per_s = ops / (best * 1e-3);
    const double bytes = mode == 0 ? 32.0 : (mode == 3 || mode == 6) ? 64.0 : 16.0;  // atomics: 8-B read + 8-B write
    printf("{\"probe\": \"%s\", \"ops_per_s\": %.4e, \"gb_s\": %.1f, \"ms\": %.3f, \"sms\": %d, \"working_set_mib\": 96}\n",
           names[mode], per_s, per_s * bytes / 1e9, best, sms);
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    fprintf(stderr, "%s\n", cudaGetErrorString(err));
    return 1;
  }
  return 0;
}
