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

// FP64 tensor-core throughput: mma.sync m8n8k4 f64 (256 FMA per warp instruction),
// 8 independent accumulator tiles per warp.  With dfma_too, the same warps also run 8
// DFMA chains per iteration to see whether the two pipes overlap.
template <bool DFMA_TOO>
__global__ void __launch_bounds__(256) k_dmma_peak(double* out, int iters, double a0, double b0) {
  double c[8][2];
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    c[j][0] = c[j][1] = 0.0;
    r[j] = threadIdx.x * 1e-3 + j;
  }
  const double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1])
                   : "d"(a), "d"(b));
      if (DFMA_TOO) r[j] = fma(r[j], a, b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + r[j];
  if (s == 1234.5) out[blockIdx.x] = s;
}

double measure_fp64_peak(cudaStream_t s);

void measure_fp64_tensor(cudaStream_t s, double* dmma_tflops, double* mixed_tflops) {
  int dev = 0, sms = 0;
  GSGPC_CUDA(cudaGetDevice(&dev));
  GSGPC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out = nullptr;
  GSGPC_CUDA(cudaMalloc(&out, sizeof(double) * sms * 8));
  const int blocks = sms * 8, iters = 2048;
  cudaEvent_t e0, e1;
  GSGPC_CUDA(cudaEventCreate(&e0));
  GSGPC_CUDA(cudaEventCreate(&e1));
  for (int mode = 0; mode < 2; ++mode) {
    double best = 0.0;
    for (int rep = 0; rep < 4; ++rep) {
      GSGPC_CUDA(cudaEventRecord(e0, s));
      if (mode == 0) k_dmma_peak<false><<<blocks, 256, 0, s>>>(out, iters, 1e-3, 1e-3);
      else k_dmma_peak<true><<<blocks, 256, 0, s>>>(out, iters, 1e-3, 1e-3);
      GSGPC_CUDA(cudaEventRecord(e1, s));
      GSGPC_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      GSGPC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      const double warps = static_cast<double>(blocks) * 8.0;
      double flops = 2.0 * 256.0 * 8.0 * iters * warps;  // DMMA
      if (mode == 1) flops += 2.0 * 8.0 * iters * warps * 32.0;  // + DFMA
      if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    if (mode == 0) *dmma_tflops = best;
    else *mixed_tflops = best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
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
