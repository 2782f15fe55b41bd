// gridsync_bench.cu — cost of one grid-wide barrier in a persistent cooperative kernel
// (the EFCG kernel runs 4 per iteration): cooperative_groups grid.sync() versus a
// single-counter barrier (one relaxed atomic per block + acquire spin on a generation word).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/gridsync_bench tools/gridsync_bench.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>

namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned long long* sink) {
  cg::grid_group grid = cg::this_grid();
  unsigned long long acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x ^ i;
    grid.sync();
  }
  if (acc == 12345) *sink = acc;
}

struct Bar {
  unsigned int count;
  unsigned int gen;
};

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_bar(Bar* b, unsigned nblocks, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned my = gen;
    __threadfence();
    const unsigned arrived = atomicAdd(&b->count, 1u) + 1;
    if (arrived == nblocks) {
      b->count = 0;
      __threadfence();
      atomicExch(&b->gen, my + 1);
    } else {
      while (ld_acq(&b->gen) == my) {
      }
    }
    gen = my + 1;
  }
  __syncthreads();
}

__global__ void k_custom(int iters, Bar* b, unsigned long long* sink) {
  __shared__ unsigned gen;
  if (threadIdx.x == 0) gen = 0;
  __syncthreads();
  unsigned g = 0;
  unsigned long long acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x ^ i;
    grid_bar(b, gridDim.x, g);
  }
  if (acc == 12345) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* sink;
  Bar* bar;
  cudaMalloc(&sink, 8);
  cudaMalloc(&bar, sizeof(Bar));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  for (int per : {1, 2}) {
    const int nb = sms * per;
    for (int kind = 0; kind < 2; ++kind) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(bar, 0, sizeof(Bar));
        int it = iters;
        void* args_cg[] = {&it, &sink};
        void* args_cu[] = {&it, &bar, &sink};
        cudaEventRecord(e0);
        if (kind == 0)
          cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_cg), nb, 256, args_cg, 0, 0);
        else
          cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_custom), nb, 256, args_cu, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      const cudaError_t err = cudaGetLastError();
      std::printf("blocks %4d %-22s %.3f us per barrier (%s)\n", nb, kind == 0 ? "cg::grid.sync" : "counter barrier",
                  1e3 * best / iters, cudaGetErrorString(err));
    }
  }
  return 0;
}
