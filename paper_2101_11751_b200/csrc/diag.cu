// diag.cu — FP64 FMA throughput microbenchmark (the precompute's FP64 roofline denominator).
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.cuh"

namespace gsgpc {

// 16 independent DFMA chains per thread, register resident; result written so the loop
// is not eliminated.
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double a, double b) {
  double r[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) r[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) r[j] = fma(r[j], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += r[j];
  if (s == 1234.5) out[blockIdx.x] = s;
}

double measure_fp64_peak(cudaStream_t s) {
  int dev = 0, sms = 0;
  GSGPC_CUDA(cudaGetDevice(&dev));
  GSGPC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out = nullptr;
  GSGPC_CUDA(cudaMalloc(&out, sizeof(double) * sms * 8));
  const int blocks = sms * 8, iters = 4096;
  cudaEvent_t e0, e1;
  GSGPC_CUDA(cudaEventCreate(&e0));
  GSGPC_CUDA(cudaEventCreate(&e1));
  k_dfma_peak<<<blocks, 256, 0, s>>>(out, iters, 0.999999, 1e-7);  // warm-up
  double best = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    GSGPC_CUDA(cudaEventRecord(e0, s));
    k_dfma_peak<<<blocks, 256, 0, s>>>(out, iters, 0.999999, 1e-7);
    GSGPC_CUDA(cudaEventRecord(e1, s));
    GSGPC_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    GSGPC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    const double flops = 2.0 * 16.0 * iters * static_cast<double>(blocks) * 256.0;
    best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return best;
}

}  // namespace gsgpc
