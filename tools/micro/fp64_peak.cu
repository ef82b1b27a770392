// FP64 pipe peak probe: independent DFMA chains, 8 per thread, all SMs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_chains(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) s += x[k];
  if (s == 12345.0) out[0] = s;
}

__global__ void dadd_chains(double* out, int iters, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = x[k] + b;
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) s += x[k];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 20000, block = 256, grid = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int kind = 0; kind < 2; kind++) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
      cudaEventRecord(e0);
      if (kind == 0) dfma_chains<<<grid, block>>>(out, iters, 0.999999, 1e-7);
      else dadd_chains<<<grid, block>>>(out, iters, 1e-7);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double ops = (double)grid * block * iters * 8;
    printf("{\"op\": \"%s\", \"instr_per_s\": %.4e, \"flops\": %.4e, \"ms\": %.3f, \"sms\": %d}\n",
           kind == 0 ? "DFMA" : "DADD", ops / (best * 1e-3), ops * (kind == 0 ? 2 : 1) / (best * 1e-3), best, sms);
  }
  return 0;
}
