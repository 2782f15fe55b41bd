// internal.cuh — shared device/host definitions of libgsgpc (B200 / sm_100a).
//
// The interpolation arithmetic here is the bit-exact restatement of the reference's
// stencil_1d / cubic_weight / linear_weight (/root/reference/proj/src/interp.cpp:27-75):
// explicit __d*_rn intrinsics forbid FMA contraction, so weights and stencil start
// indices equal the reference's (g++ -O3 without -march emits no FMA) bit for bit.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <stdexcept>
#include <utility>
#include <string>

#include "../../include/gsgpc.h"

namespace gsgpc {

// ------------------------------------------------------------------ errors (host)
struct Error : std::runtime_error {
  gsgpc_status code;
  int64_t row;
  Error(gsgpc_status c, const std::string& m, int64_t r = 0) : std::runtime_error(m), code(c), row(r) {}
};

#define GSGPC_CUDA(expr)                                                                   \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess) {                                                               \
      throw ::gsgpc::Error(GSGPC_CUDA_ERROR, std::string(#expr " failed: ") +              \
                                                 cudaGetErrorString(_e));                  \
    }                                                                                      \
  } while (0)

inline void invalid(const std::string& m) { throw Error(GSGPC_INVALID_ARGUMENT, m); }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-device property of a kernel: keep
// what was set per (device, kernel), under a lock, so every device (and every thread) sees
// the attribute before its first launch needing it.
// Streaming multiprocessors of the current device (148 on B200), cached per device.
inline int sm_count() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
  cache[dev] = n;
  return n;
}

inline void set_max_dynamic_smem(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  GSGPC_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  int& cur = done[{dev, func}];
  if (bytes <= cur || bytes <= 48 * 1024) return;
  GSGPC_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  cur = bytes;
}

// ------------------------------------------------------------------ grid descriptor
struct GridDev {
  int d;
  int W;                  // stencil width per dimension: 4 cubic, 2 linear
  double mn[GSGPC_MAX_DIM];
  double sp[GSGPC_MAX_DIM];
  double isp[GSGPC_MAX_DIM];     // 1 / spacing (fast classification path)
  int64_t sz[GSGPC_MAX_DIM];     // nodes per dimension
  int64_t nc[GSGPC_MAX_DIM];     // cells per dimension = sz - 1
  int64_t m;              // Π sz
  int64_t cells;          // Π nc
};

// Point source descriptor (see gsgpc_points).
struct PointsDev {
  const void* x;
  const void* y;
  int64_t xs;                    // row stride (elements)
  int64_t xo[GSGPC_MAX_DIM];     // column offsets (elements)
  int64_t ys;
};

// ------------------------------------------------------------------ interp math (device)
// Point classification.  Order mirrors the reference: stencil_1d() runs for every
// dimension first (an out-of-range u throws "point outside grid", interp.cpp:53-55), then
// the tensor-product loop (interp.cpp:101-130) visits dimensions in order: a NaN
// coordinate yields all-zero weights (the combo loop breaks on a zero weight and the
// point contributes nothing), an out-of-range stencil node with a nonzero weight throws
// "stencil leaves the grid".
enum : int { PT_VALID = 0, PT_OUTSIDE = 1, PT_LEAVES = 2, PT_EMPTY = 3 };

__device__ __forceinline__ double cubic_w(double tt) {
  const double a = fabs(tt);
  if (a <= 1.0) return __dadd_rn(__dmul_rn(__dmul_rn(__dsub_rn(__dmul_rn(1.5, a), 2.5), a), a), 1.0);
  if (a < 2.0) {
    return __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(__dadd_rn(__dmul_rn(-0.5, a), 2.5), a), 4.0), a), 2.0);
  }
  return 0.0;
}
__device__ __forceinline__ double linear_w(double tt) {
  const double a = fabs(tt);
  return a <= 1.0 ? __dsub_rn(1.0, a) : 0.0;
}

// stencil_1d (interp.cpp:45-75): u, snap, range check, i0 clamp, t.
// Returns PT_VALID / PT_OUTSIDE / PT_EMPTY (NaN u).
__device__ __forceinline__ int stencil_dim(double x, double mn, double sp, int64_t size, int64_t& i0,
                                           double& t) {
  double u = __ddiv_rn(__dsub_rn(x, mn), sp);
  const double r = round(u);
  if (fabs(__dsub_rn(u, r)) < 1e-9) u = r;
  if (u < 0.0 || u > static_cast<double>(size - 1)) return PT_OUTSIDE;
  if (u != u) return PT_EMPTY;
  int64_t i = static_cast<int64_t>(floor(u));
  if (i > size - 2) i = size - 2;
  i0 = i;
  t = __dsub_rn(u, static_cast<double>(i));
  return PT_VALID;
}

// Same result as stencil_dim (status, cell index i0; t to within a few ulp) without the
// IEEE division on all but a measure-zero set of inputs.  u ≈ (x - min)·(1/spacing)
// differs from the correctly rounded quotient u* by ≤ 2 ulp(u) ≤ |u|·2^-51.  With
// d = |u - round(u)| and margin e = 1e-12 + |u|·2^-48:
//   d < 1e-9 - e  → |u* - round(u*)| < 1e-9: the reference snaps, u = round(u) exactly;
//   d > 1e-9 + e  → it does not snap, and floor(u) = floor(u*) (no integer in between) and
//                   the range tests agree;
//   otherwise (|d - 1e-9| ≤ e) → fall back to the exact division.
// NaN / ±inf take the first branch with u = NaN / ±inf and classify like stencil_dim.
// Used by the precompute (cell binning + moments, tolerance 1e-10), never for reported weights.
__device__ __forceinline__ int stencil_dim_fast(double x, double mn, double sp, double isp, int64_t size,
                                                int64_t& i0, double& t) {
  double u = __dsub_rn(x, mn) * isp;
  const double r = round(u);
  const double dd = fabs(u - r);
  const double e = 1e-12 + fabs(u) * 3.552713678800501e-15;
  if (dd >= 1e-9 - e && dd <= 1e-9 + e) return stencil_dim(x, mn, sp, size, i0, t);
  if (dd < 1e-9) u = r;
  if (u < 0.0 || u > static_cast<double>(size - 1)) return PT_OUTSIDE;
  if (u != u) return PT_EMPTY;
  int64_t i = static_cast<int64_t>(floor(u));
  if (i > size - 2) i = size - 2;
  i0 = i;
  t = u - static_cast<double>(i);
  return PT_VALID;
}

// 1-D weights in the reference order (cubic: start i0-1, [c(t+1), c(t), c(1-t), c(2-t)];
// linear: start i0, [l(t), l(1-t)]).
__device__ __forceinline__ void weights_1d(double t, int W, double* w) {
  if (W == 4) {
    w[0] = cubic_w(__dadd_rn(t, 1.0));
    w[1] = cubic_w(t);
    w[2] = cubic_w(__dsub_rn(1.0, t));
    w[3] = cubic_w(__dsub_rn(2.0, t));
  } else {
    w[0] = linear_w(t);
    w[1] = linear_w(__dsub_rn(1.0, t));
  }
}

// Does the 1-D stencil of (i0, t) put a nonzero weight on a node outside [0, size)?
__device__ __forceinline__ bool leaves_dim(int64_t i0, double t, int64_t size, int W) {
  if (W != 4) return false;  // linear: start i0 >= 0, i0 + 1 <= size - 1 always
  if (i0 == 0 && cubic_w(__dadd_rn(t, 1.0)) != 0.0) return true;       // node i0-1 = -1
  if (i0 + 2 >= size && cubic_w(__dsub_rn(2.0, t)) != 0.0) return true;  // node i0+2 = size
  return false;
}

template <typename T>
__device__ __forceinline__ void load_point(const PointsDev& p, int d, int64_t i, double* x, double& y) {
  const T* X = static_cast<const T*>(p.x);
  const T* Y = static_cast<const T*>(p.y);
#pragma unroll
  for (int k = 0; k < GSGPC_MAX_DIM; ++k) {
    if (k < d) x[k] = static_cast<double>(X[i * p.xs + p.xo[k]]);
  }
  y = static_cast<double>(Y[i * p.ys]);
}

// Full classification of one point; on PT_VALID fills i0[k], t[k] and the cell id.
__device__ __forceinline__ int classify(const GridDev& g, const double* x, int64_t* i0, double* t,
                                        int64_t& cell) {
  int st[GSGPC_MAX_DIM];
#pragma unroll
  for (int k = 0; k < GSGPC_MAX_DIM; ++k) {
    if (k < g.d) {
      st[k] = stencil_dim_fast(x[k], g.mn[k], g.sp[k], g.isp[k], g.sz[k], i0[k], t[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < GSGPC_MAX_DIM; ++k) {
    if (k < g.d && st[k] == PT_OUTSIDE) return PT_OUTSIDE;
  }
#pragma unroll
  for (int k = 0; k < GSGPC_MAX_DIM; ++k) {
    if (k < g.d) {
      if (st[k] == PT_EMPTY) return PT_EMPTY;
      if (leaves_dim(i0[k], t[k], g.sz[k], g.W)) return PT_LEAVES;
    }
  }
  int64_t c = 0;
#pragma unroll
  for (int k = 0; k < GSGPC_MAX_DIM; ++k) {
    if (k < g.d) c = c * g.nc[k] + i0[k];
  }
  cell = c;
  return PT_VALID;
}

// ------------------------------------------------------------------ misc device helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh /*NT/32*/) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = l < NT / 32 ? sh[l] : 0.0;
    r = warp_sum(r);
  }
  return r;  // valid in thread 0
}

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace gsgpc
