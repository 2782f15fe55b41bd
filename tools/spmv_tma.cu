// spmv_tma.cu — diagnostic microbenchmark (not part of the library): the config-3 half-stencil
// SpMV (80×80×20 grid, S_min = 172, offset-major A[s][node]) two ways:
//   ldg : the library's stencil_row_dot (8 offsets of loads in flight per thread)
//   tma : a producer warp streams each 256-node tile's stencil rows (forward A[s][a] and
//         mirrored A[s][a − o_s]) into a shared-memory ring with cp.async.bulk + mbarriers;
//         256 consumer threads read them from shared memory (v through L1).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2101_11751_b200/csrc \
//        -o tools/_spmv_tma tools/spmv_tma.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

#include "stencil_spmv.cuh"

using namespace gsgpc;

constexpr int SMIN = 172;
__constant__ int c_off[SMIN];
struct Off {
  __device__ __forceinline__ int operator()(int s) const { return c_off[s]; }
};

__global__ void __launch_bounds__(256) k_ldg(int m, const double* __restrict__ A, const double* __restrict__ v,
                                             double* __restrict__ out) {
  for (int a = blockIdx.x * 256 + threadIdx.x; a < m; a += gridDim.x * 256)
    out[a] = stencil_row_dot<SMIN>(m, A, v, a, Off{});
}

// ---------------------------------------------------------------- TMA ring
constexpr int TN = 256;             // nodes per tile (one per consumer thread)
constexpr int TU = 4;               // offsets per stage
constexpr int TB = TN + 4;          // mirrored row window (even-aligned start)
constexpr int NG = (SMIN - 1 + TU - 1) / TU;  // 43 groups for s = 1..171
constexpr int STAGE_DBL = TU * (TN + TB);

__device__ __forceinline__ unsigned sa(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}\n" ::"r"(sa(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
               "l"(src), "r"(bytes), "r"(sa(bar))
               : "memory");
}

__device__ __forceinline__ int bwd_start(int base, int o) {
  const int b = base - o;
  return b < 0 ? 0 : (b & ~1);
}

template <int S>
__global__ void __launch_bounds__(288) k_tma(int m, const double* __restrict__ A, const double* __restrict__ v,
                                             double* __restrict__ out) {
  extern __shared__ __align__(128) double ring[];  // S stages × STAGE_DBL
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int ntiles = (m + TN - 1) / TN;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], TN / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= TN) {  // producer warp
    if (threadIdx.x != TN) return;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int base = tile * TN;
      const int nn = min(TN, m - base);
      const unsigned fbytes = static_cast<unsigned>(((nn + 1) & ~1) * 8);
      for (int gI = 0; gI < NG; ++gI, ++it) {
        const int st = it % S;
        mbar_wait(&empty[st], ((it / S) & 1) ^ 1);
        double* buf = ring + st * STAGE_DBL;
        const int nq = min(TU, SMIN - 1 - gI * TU);
        mbar_expect(&full[st], static_cast<unsigned>(nq) * (fbytes + TB * 8));
        for (int q = 0; q < nq; ++q) {
          const int s = 1 + gI * TU + q;
          const double* row = A + static_cast<int64_t>(s) * m;
          bulk_g2s(buf + q * TN, row + base, fbytes, &full[st]);
          bulk_g2s(buf + TU * TN + q * TB, row + bwd_start(base, c_off[s]), TB * 8, &full[st]);
        }
      }
    }
    return;
  }
  // consumers
  const int t = threadIdx.x;
  int it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int base = tile * TN;
    const int a = base + t;
    const bool live = a < m;
    double acc0 = live ? __ldg(A + a) * __ldca(v + a) : 0.0, acc1 = 0.0;
    for (int gI = 0; gI < NG; ++gI, ++it) {
      const int st = it % S;
      mbar_wait(&full[st], (it / S) & 1);
      const double* buf = ring + st * STAGE_DBL;
#pragma unroll
      for (int q = 0; q < TU; ++q) {
        const int s = 1 + gI * TU + q;
        if (s < SMIN && live) {
          const int o = c_off[s];
          const int f = a + o, b = a - o;
          if (static_cast<unsigned>(f) < static_cast<unsigned>(m)) acc0 = fma(buf[q * TN + t], __ldca(v + f), acc0);
          if (b >= 0) acc1 = fma(buf[TU * TN + q * TB + (b - bwd_start(base, o))], __ldca(v + b), acc1);
        }
      }
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(&empty[st]);
    }
    if (live) out[a] = acc0 + acc1;
  }
}

// ---------------------------------------------------------------- TMA ring, lane-parallel issue
// Same ring, but the producer warp issues the 2·TU2 bulk copies of a stage from 2·TU2 lanes at
// once (one copy per lane) instead of one thread issuing them in turn.
template <int TU2, int S>
__global__ void __launch_bounds__(288) k_tma2(int m, const double* __restrict__ A, const double* __restrict__ v,
                                              double* __restrict__ out) {
  static_assert(2 * TU2 <= 32, "one copy per producer lane");
  constexpr int NG2 = (SMIN - 1 + TU2 - 1) / TU2;
  constexpr int STG = TU2 * (TN + TB);
  extern __shared__ __align__(128) double ring[];
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int ntiles = (m + TN - 1) / TN;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], TN / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= TN) {  // producer warp
    const int lane = threadIdx.x - TN;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int base = tile * TN;
      const int nn = min(TN, m - base);
      const unsigned fbytes = static_cast<unsigned>(((nn + 1) & ~1) * 8);
      for (int gI = 0; gI < NG2; ++gI, ++it) {
        const int st = it % S;
        if (lane == 0) mbar_wait(&empty[st], ((it / S) & 1) ^ 1);
        __syncwarp();
        double* buf = ring + st * STG;
        const int nq = min(TU2, SMIN - 1 - gI * TU2);
        if (lane == 0) mbar_expect(&full[st], static_cast<unsigned>(nq) * (fbytes + TB * 8));
        __syncwarp();
        const int q = lane >> 1, dir = lane & 1;
        if (q < nq) {
          const int s = 1 + gI * TU2 + q;
          const double* row = A + static_cast<int64_t>(s) * m;
          if (dir == 0) bulk_g2s(buf + q * TN, row + base, fbytes, &full[st]);
          else bulk_g2s(buf + TU2 * TN + q * TB, row + bwd_start(base, c_off[s]), TB * 8, &full[st]);
        }
      }
    }
    return;
  }
  const int t = threadIdx.x;
  int it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int base = tile * TN;
    const int a = base + t;
    const bool live = a < m;
    double acc0 = live ? __ldg(A + a) * __ldca(v + a) : 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    for (int gI = 0; gI < NG2; ++gI, ++it) {
      const int st = it % S;
      // v loads do not depend on the ring: issue them before waiting for the stage
      double vf[TU2], vb[TU2];
      int bo[TU2];
#pragma unroll
      for (int q = 0; q < TU2; ++q) {
        const int s = 1 + gI * TU2 + q;
        const int o = s < SMIN ? c_off[s] : 0;
        const int f = a + o, b = a - o;
        const bool okf = live && s < SMIN && static_cast<unsigned>(f) < static_cast<unsigned>(m);
        const bool okb = live && s < SMIN && b >= 0;
        vf[q] = okf ? __ldca(v + f) : 0.0;
        vb[q] = okb ? __ldca(v + b) : 0.0;
        bo[q] = okb ? b - bwd_start(base, o) : 0;
      }
      mbar_wait(&full[st], (it / S) & 1);
      const double* buf = ring + st * STG;
#pragma unroll
      for (int q = 0; q < TU2; q += 2) {
        acc0 = fma(buf[q * TN + t], vf[q], acc0);
        acc1 = fma(buf[TU2 * TN + q * TB + bo[q]], vb[q], acc1);
        if (q + 1 < TU2) {
          acc2 = fma(buf[(q + 1) * TN + t], vf[q + 1], acc2);
          acc3 = fma(buf[TU2 * TN + (q + 1) * TB + bo[q + 1]], vb[q + 1], acc3);
        }
      }
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(&empty[st]);
    }
    if (live) out[a] = (acc0 + acc1) + (acc2 + acc3);
  }
}

int main() {
  const int n0 = 80, n1 = 80, n2 = 20, m = n0 * n1 * n2;
  std::vector<int> off;
  for (int s = 0; s < SMIN; ++s) {
    int q = 171 + s, d[3];
    for (int k = 2; k >= 0; --k) {
      d[k] = q % 7 - 3;
      q /= 7;
    }
    off.push_back((d[0] * n1 + d[1]) * n2 + d[2]);
  }
  cudaMemcpyToSymbol(c_off, off.data(), sizeof(int) * SMIN);
  std::vector<double> hA(static_cast<size_t>(SMIN) * m + 64), hv(m);
  unsigned long long x = 88172645463325252ull;
  auto rnd = [&] {
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    return (x >> 11) * 0x1.0p-53;
  };
  for (auto& e : hA) e = rnd();
  for (auto& e : hv) e = rnd() - 0.5;
  double *A, *v, *o1, *o2, *flush;
  const size_t fl = size_t(512) << 20;
  cudaMalloc(&A, sizeof(double) * hA.size());
  cudaMalloc(&v, sizeof(double) * m);
  cudaMalloc(&o1, sizeof(double) * m);
  cudaMalloc(&o2, sizeof(double) * m);
  cudaMalloc(&flush, fl);
  cudaMemcpy(A, hA.data(), sizeof(double) * hA.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(v, hv.data(), sizeof(double) * m, cudaMemcpyHostToDevice);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int cold = 0; cold < 2; ++cold) {
      float best = 1e30f, sum = 0.0f;
      const int reps = 30;
      for (int r = 0; r < reps; ++r) {
        if (cold) cudaMemsetAsync(flush, r, fl);
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
        sum += ms;
      }
      std::printf("%-34s %s  best %6.1f us  mean %6.1f us  %s\n", name, cold ? "cold" : "warm", best * 1e3,
                  sum / reps * 1e3, cudaGetErrorString(cudaGetLastError()));
    }
  };
  run("ldg grid 2/SM", [&] { k_ldg<<<2 * sms, 256>>>(m, A, v, o1); });
  run("ldg node/thread", [&] { k_ldg<<<(m + 255) / 256, 256>>>(m, A, v, o1); });
  auto tma = [&](auto kern, int S, int per_sm, const char* name) {
    const size_t smem = sizeof(double) * S * STAGE_DBL;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    run(name, [&] { kern<<<per_sm * sms, 288, smem>>>(m, A, v, o2); });
    std::vector<double> r1(m), r2(m);
    cudaMemcpy(r1.data(), o1, sizeof(double) * m, cudaMemcpyDeviceToHost);
    cudaMemcpy(r2.data(), o2, sizeof(double) * m, cudaMemcpyDeviceToHost);
    double err = 0.0, mx = 0.0;
    for (int i = 0; i < m; ++i) {
      err = std::max(err, std::abs(r1[i] - r2[i]));
      mx = std::max(mx, std::abs(r1[i]));
    }
    std::printf("    max |tma - ldg| = %.3g (max |y| %.3g)\n", err, mx);
  };
  tma(k_tma<4>, 4, 2, "tma S=4 2/SM");
  tma(k_tma<6>, 6, 2, "tma S=6 2/SM");
  tma(k_tma<8>, 8, 1, "tma S=8 1/SM");
  tma(k_tma<12>, 12, 1, "tma S=12 1/SM");
  tma(k_tma<4>, 4, 3, "tma S=4 3/SM");
  auto tma2 = [&](auto kern, int TU2, int S, int per_sm, const char* name) {
    const size_t smem = sizeof(double) * S * TU2 * (TN + TB);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    run(name, [&] { kern<<<per_sm * sms, 288, smem>>>(m, A, v, o2); });
    std::vector<double> r1(m), r2(m);
    cudaMemcpy(r1.data(), o1, sizeof(double) * m, cudaMemcpyDeviceToHost);
    cudaMemcpy(r2.data(), o2, sizeof(double) * m, cudaMemcpyDeviceToHost);
    double err = 0.0;
    for (int i = 0; i < m; ++i) err = std::max(err, std::abs(r1[i] - r2[i]));
    std::printf("    max |tma2 - ldg| = %.3g\n", err);
  };
  tma2(k_tma2<4, 6>, 4, 6, 2, "tma2 TU=4 S=6 2/SM");
  tma2(k_tma2<8, 3>, 8, 3, 2, "tma2 TU=8 S=3 2/SM");
  tma2(k_tma2<8, 6>, 8, 6, 1, "tma2 TU=8 S=6 1/SM");
  tma2(k_tma2<8, 4>, 8, 4, 1, "tma2 TU=8 S=4 1/SM");
  tma2(k_tma2<16, 3>, 16, 3, 1, "tma2 TU=16 S=3 1/SM");
  tma2(k_tma2<4, 4>, 4, 4, 3, "tma2 TU=4 S=4 3/SM");
  tma2(k_tma2<8, 2>, 8, 2, 3, "tma2 TU=8 S=2 3/SM");
  tma2(k_tma2<4, 3>, 4, 3, 4, "tma2 TU=4 S=3 4/SM");
  return 0;
}
