// efla.cu — probe-batched factorized Lanczos (EFLA, factorized_lanczos_fused,
// solvers.cpp:464-538) and the SLQ log-likelihood (log_likelihood_gsgp SkiOperator route,
// gp.cpp:158-240 with slq_logdet_ski_factorized, gp.cpp:85-111).
//
// All P probes advance together: one stencil read per step serves every probe (K6 SpMM),
// the K_G mode products treat the probe index as an extra outer dimension, and the full
// reorthogonalisation is a pair of batched GEMVs against the stored Q̂ / P̂ columns.
// Per-probe scalars (c_q, e, β_prev, scale, breakdown) stay on the device; vectors are
// probe-major [P][m].  Dots reduce through fixed per-block partials (deterministic).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <random>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/gsgpc.h"
#include "internal.cuh"
#include "precompute.cuh"

namespace gsgpc {
namespace cg = cooperative_groups;

constexpr int EF_NT = 256;
constexpr int EF_MAXP = 32;

struct EfScal {
  double cq, cqp, bprev, e, alpha, scale, b;
  int done, order;
};

// --------------------------------------------------------------- generic batched pieces
// dots: out partials [P][nd][nblk] of Σ_a x_k[p][a]·y_k[p][a]
struct DotSpec {
  const double* x[6];
  const double* y[6];
  int nd;
};

__device__ __forceinline__ void block_partial_store(double v, double* dst, double* sh) {
  const double s = block_sum<EF_NT>(v, sh);
  if (threadIdx.x == 0) *dst = s;
}

// wv = sbar + cq·kwt - bprev·qprev;  dots pcur·wv, wv·wt
__global__ void __launch_bounds__(EF_NT) k_ef_s1(int64_t m, const EfScal* sc, const double* sbar, const double* kwt,
                                                 const double* qprev, double* wv, const double* pcur, const double* wt,
                                                 double* part, int nblk) {
  __shared__ double sh[8];
  const int p = blockIdx.y;
  const EfScal s = sc[p];
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  double d0 = 0.0, d1 = 0.0;
  if (!s.done && a < m) {
    const int64_t o = static_cast<int64_t>(p) * m + a;
    const double w = sbar[o] + s.cq * kwt[o] - s.bprev * qprev[o];
    wv[o] = w;
    d0 = pcur[o] * w;
    d1 = w * wt[o];
  }
  block_partial_store(d0, part + (static_cast<int64_t>(p) * 2 + 0) * nblk + blockIdx.x, sh);
  block_partial_store(d1, part + (static_cast<int64_t>(p) * 2 + 1) * nblk + blockIdx.x, sh);
}

// reduce partials [R][nblk] → out[R]
__global__ void __launch_bounds__(EF_NT) k_ef_reduce(const double* part, int nblk, double* out) {
  __shared__ double sh[8];
  const int r = blockIdx.x;
  double v = 0.0;
  for (int i = threadIdx.x; i < nblk; i += EF_NT) v += part[static_cast<int64_t>(r) * nblk + i];
  const double s = block_sum<EF_NT>(v, sh);
  if (threadIdx.x == 0) out[r] = s;
}

// alpha_i (solvers.cpp:494-500)
__global__ void k_ef_c1(int P, int i, int k, double s2, EfScal* sc, const double* dots /*P×2*/, const double* tq,
                        double* alpha) {
  const int p = threadIdx.x;
  if (p >= P) return;
  EfScal s = sc[p];
  if (s.done) return;
  s.e = s2 * s.cq - s.bprev * s.cqp;
  const double al = dots[p * 2 + 0] + s.e * tq[p * k + i] + s.cq * dots[p * 2 + 1] + s.cq * s.e;
  alpha[p * k + i] = al;
  s.alpha = al;
  s.scale = fmax(s.scale, fabs(al));
  if (i == k - 1) {
    s.order = k;
  } else {
    s.e -= al * s.cq;
  }
  sc[p] = s;
}

// wv -= alpha·q; partials of wv·wt and P̂_j·wv (j ≤ i).  The i + 2 block sums run as one pass:
// each warp reduces its values per j with shuffles into wsum[warp][j] (the P̂_j loads issued 8
// at a time), one barrier, then thread j adds the 8 warp partials of column j — instead of
// i + 2 block_sum calls with two barriers each (0.85 ms per Lanczos step at config 5).
constexpr int EF_MAXK = 256;  // Lanczos depth bound of the one-pass reduction (shared memory)

__device__ __forceinline__ double ef_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(EF_NT) k_ef_s2(int64_t m, int i, int k, const EfScal* sc, double* wv, const double* q,
                                                 const double* wt, const double* Ph, double* part, int nblk) {
  __shared__ double wsum[EF_NT / 32][EF_MAXK];
  const int p = blockIdx.y;
  const EfScal s = sc[p];
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  const int nd = i + 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double w = 0.0;
  const bool live = !s.done && a < m;
  const int64_t o = static_cast<int64_t>(p) * m + a;
  if (live) {
    w = wv[o] - s.alpha * q[o];
    wv[o] = w;
  }
  const double w0 = live ? w * wt[o] : 0.0;
  const double* ph = Ph + static_cast<int64_t>(p) * k * m + a;
  // columns c = 0 (wv·wt) and c = 1 + j (P̂_j·wv), EF_MAXK columns per pass
  for (int c0 = 0; c0 < nd; c0 += EF_MAXK) {
    const int c1 = min(nd, c0 + EF_MAXK);
    for (int cb = c0; cb < c1; cb += 8) {
      double t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = cb + u;
        t[u] = (live && c < c1) ? (c == 0 ? w0 : ph[static_cast<int64_t>(c - 1) * m] * w) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double r = ef_warp_sum(t[u]);
        if (lane == 0 && cb + u < c1) wsum[warp][cb + u - c0] = r;
      }
    }
    __syncthreads();
    for (int c = c0 + threadIdx.x; c < c1; c += EF_NT) {
      double r = 0.0;
#pragma unroll
      for (int ww = 0; ww < EF_NT / 32; ++ww) r += wsum[ww][c - c0];
      part[(static_cast<int64_t>(p) * nd + c) * nblk + blockIdx.x] = r;
    }
    __syncthreads();
  }
}

// λ_j = P̂_j·wv + e·tq_j + (wv·wt + e)·d_j ; e -= d·λ   (solvers.cpp:505-509)
__global__ void k_ef_c2(int P, int i, int k, EfScal* sc, const double* dots /*P×(i+2)*/, const double* tq,
                        const double* dv, double* lam) {
  const int p = threadIdx.x;
  if (p >= P) return;
  EfScal s = sc[p];
  if (s.done) return;
  const int nd = i + 2;
  const double wdot = dots[p * nd + 0];
  double dl = 0.0;
  for (int j = 0; j <= i; ++j) {
    const double l = dots[p * nd + 1 + j] + s.e * tq[p * k + j] + (wdot + s.e) * dv[p * k + j];
    lam[p * k + j] = l;
    dl += dv[p * k + j] * l;
  }
  s.e -= dl;
  sc[p] = s;
}

// wv -= Σ_j Q̂_j λ_j
__global__ void __launch_bounds__(EF_NT) k_ef_g2(int64_t m, int i, int k, const EfScal* sc, double* wv, const double* Qh,
                                                 const double* lam) {
  const int p = blockIdx.y;
  if (sc[p].done) return;
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  if (a >= m) return;
  double acc = 0.0;
  for (int j = 0; j <= i; ++j) acc += Qh[(static_cast<int64_t>(p) * k + j) * m + a] * lam[p * k + j];
  wv[static_cast<int64_t>(p) * m + a] -= acc;
}

// Batched stencil SpMV: out[p] = W^T W x[p] for P ≤ 32 probes; each stencil value is read
// once and applied to every probe.
template <int PB, int SMIN>
__global__ void __launch_bounds__(128) k_spmm(int64_t m, const double* __restrict__ A, const double* __restrict__ x,
                                              double* __restrict__ out, int P, const EfScal* sc,
                                              const __grid_constant__ StencilOffsets off) {
  const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= m) return;
  double acc[PB];
  const double a0 = A[a];
#pragma unroll
  for (int p = 0; p < PB; ++p) acc[p] = p < P ? a0 * x[p * m + a] : 0.0;
  // check-free: off-grid partners hit exactly-zero stencil entries (see operators.cu)
#pragma unroll 2
  for (int s = 1; s < SMIN; ++s) {
    const int64_t o = off.flat[s];
    const int64_t f = a + o, b = a - o;
    if (f >= 0 && f < m) {
      const double v = A[s * m + a];
#pragma unroll
      for (int p = 0; p < PB; ++p)
        if (p < P) acc[p] = fma(v, x[p * m + f], acc[p]);
    }
    if (b >= 0 && b < m) {
      const double v = A[s * m + b];
#pragma unroll
      for (int p = 0; p < PB; ++p)
        if (p < P) acc[p] = fma(v, x[p * m + b], acc[p]);
    }
  }
#pragma unroll
  for (int p = 0; p < PB; ++p)
    if (p < P && !(sc && sc[p].done)) out[p * m + a] = acc[p];
}

// Batched SpMV over P right-hand sides, tiled along the last grid dimension.  The grid-stride
// version (k_spmm) read x[p][a ± o_s] for 2·S_min offsets × P vectors per node straight from
// L2 (P = 30 vectors of 2 MB do not stay in L1): ~21 GB of L2 traffic per call at config 5.
// Here a block owns T = 128 consecutive nodes; for each pencil of the full stencil (the E
// offsets that differ only in the last dimension, E^(d−1) pencils) it stages the P windows
// x[p][a0 + o_pencil − (W−1) .. + T + (W−1)) in shared memory once and every node then
// applies the pencil's E coefficients from it — x is read ~E× less from L2.  Coefficients
// come from the stored half at the node (A[s][a]) or mirrored at the partner (A[s'][a + o]);
// partners across the grid edge meet stored exact zeros (check-free, finite vectors).
constexpr int PEN_T = 128;

template <int PB, int W>
__global__ void __launch_bounds__(PEN_T) k_spmm_pencil(int m, int npen, const double* __restrict__ A,
                                                       const double* __restrict__ x, double* __restrict__ out, int P,
                                                       const EfScal* sc, const __grid_constant__ PencilTables pt) {
  constexpr int E = 2 * W - 1, WL = PEN_T + 2 * (W - 1);
  extern __shared__ double win[];  // [P][WL]
  const int a0 = blockIdx.x * PEN_T;
  const int a = a0 + threadIdx.x;
  double acc[PB];
#pragma unroll
  for (int p = 0; p < PB; ++p) acc[p] = 0.0;
  for (int q = 0; q < npen; ++q) {
    const int ob = pt.ob[q];
    __syncthreads();
    for (int i = threadIdx.x; i < P * WL; i += PEN_T) {
      const int p = i / WL, t = i - p * WL;
      const int g = a0 + ob - (W - 1) + t;
      win[i] = (g >= 0 && g < m) ? __ldcg(x + static_cast<int64_t>(p) * m + g) : 0.0;
    }
    __syncthreads();
    if (a < m) {
#pragma unroll
      for (int t = 0; t < E; ++t) {
        const int sidx = pt.s[q][t];
        const int o = ob + t - (W - 1);
        double c;
        if (sidx >= 0) {
          c = __ldg(A + static_cast<int64_t>(sidx) * m + a);
        } else {
          const int b = a + o;
          c = (b >= 0 && b < m) ? __ldg(A + static_cast<int64_t>(-sidx - 1) * m + b) : 0.0;
        }
        const double* wp = win + threadIdx.x + t;
#pragma unroll
        for (int p = 0; p < PB; ++p)
          if (p < P) acc[p] = fma(c, wp[p * WL], acc[p]);
      }
    }
  }
  if (a < m) {
#pragma unroll
    for (int p = 0; p < PB; ++p)
      if (p < P && !(sc && sc[p].done)) out[static_cast<int64_t>(p) * m + a] = acc[p];
  }
}

// Two consecutive nodes per thread and half of the probes per block (grid.y = 2): one window
// of E + 1 partners serves both nodes' E terms, read as 16-byte shared loads — 43 % fewer
// shared-memory wavefronts per FMA than one node per thread.
constexpr int PEN2_T = 128;  // threads per block (2 · 128 nodes)

template <int PH, int W>
__global__ void __launch_bounds__(PEN2_T) k_spmm_pencil2(int m, int npen, const double* __restrict__ A,
                                                         const double* __restrict__ x, double* __restrict__ out,
                                                         int P, const EfScal* sc,
                                                         const __grid_constant__ PencilTables pt) {
  constexpr int E = 2 * W - 1, NT = 2 * PEN2_T, WL = NT + 2 * (W - 1) + 2;  // even row length
  extern __shared__ __align__(16) double win2[];  // [PH][WL]
  const int p0 = blockIdx.y * PH;
  const int np = min(PH, P - p0);
  if (np <= 0) return;
  const int a0 = blockIdx.x * NT;
  const int a = a0 + 2 * threadIdx.x;
  const bool ok0 = a < m, ok1 = a + 1 < m;
  const bool vec = (m & 1) == 0;
  double acc0[PH], acc1[PH];
#pragma unroll
  for (int p = 0; p < PH; ++p) acc0[p] = acc1[p] = 0.0;
  for (int q = 0; q < npen; ++q) {
    const int ob = pt.ob[q];
    __syncthreads();
    for (int i = threadIdx.x; i < np * WL; i += PEN2_T) {
      const int p = i / WL, t = i - p * WL;
      const int g = a0 + ob - (W - 1) + t;
      win2[i] = (g >= 0 && g < m) ? __ldcg(x + static_cast<int64_t>(p0 + p) * m + g) : 0.0;
    }
    __syncthreads();
    double c0[E], c1[E];
#pragma unroll
    for (int t = 0; t < E; ++t) {
      const int sidx = pt.s[q][t];
      const int o = ob + t - (W - 1);
      c0[t] = c1[t] = 0.0;
      if (sidx >= 0) {
        const double* As = A + static_cast<int64_t>(sidx) * m;
        if (ok1 && vec) {
          const double2 cc = __ldg(reinterpret_cast<const double2*>(As + a));
          c0[t] = cc.x;
          c1[t] = cc.y;
        } else {
          c0[t] = ok0 ? __ldg(As + a) : 0.0;
          c1[t] = ok1 ? __ldg(As + a + 1) : 0.0;
        }
      } else {
        const double* As = A + static_cast<int64_t>(-sidx - 1) * m;
        const int b = a + o;
        c0[t] = (ok0 && b >= 0 && b < m) ? __ldg(As + b) : 0.0;
        c1[t] = (ok1 && b + 1 >= 0 && b + 1 < m) ? __ldg(As + b + 1) : 0.0;
      }
    }
#pragma unroll
    for (int p = 0; p < PH; ++p) {
      if (p < np) {
        const double2* wp = reinterpret_cast<const double2*>(win2 + p * WL + 2 * threadIdx.x);
        double w[E + 1];
#pragma unroll
        for (int k = 0; k < (E + 1) / 2; ++k) {
          const double2 v = wp[k];
          w[2 * k] = v.x;
          w[2 * k + 1] = v.y;
        }
#pragma unroll
        for (int t = 0; t < E; ++t) {
          acc0[p] = fma(c0[t], w[t], acc0[p]);
          acc1[p] = fma(c1[t], w[t + 1], acc1[p]);
        }
      }
    }
  }
#pragma unroll
  for (int p = 0; p < PH; ++p) {
    if (p < np && !(sc && sc[p0 + p].done)) {
      if (ok0) out[static_cast<int64_t>(p0 + p) * m + a] = acc0[p];
      if (ok1) out[static_cast<int64_t>(p0 + p) * m + a + 1] = acc1[p];
    }
  }
}

static void launch_spmm(const Launch& L, const StencilDesc& sd, const double* A, const double* x, double* out, int P,
                        const EfScal* sc) {
  static const bool grid_stride = [] {
    const char* e = getenv("GSGPC_SPMM_GRID");
    return e && e[0] == '1';
  }();
  if (!grid_stride && sd.d >= 2 && sd.m < (int64_t{1} << 31)) {
    const PencilTables pt = make_pencil_tables(sd);
    int npen = 1;
    for (int k = 0; k + 1 < sd.d; ++k) npen *= 2 * sd.W - 1;
    const unsigned blocks = static_cast<unsigned>(ceil_div(sd.m, PEN_T));
    const int WL = PEN_T + 2 * (sd.W - 1);
    const size_t smem = sizeof(double) * static_cast<size_t>(P) * WL;
    static const bool one_node = [] {
      const char* e = getenv("GSGPC_SPMM_ONE_NODE");  // diagnostics: one node per thread
      return e && e[0] == '1';
    }();
    if (sd.W == 4 && !one_node) {
      constexpr int PH = 16, WL2 = 2 * PEN2_T + 6 + 2;
      const size_t sm2 = sizeof(double) * PH * WL2;
      const dim3 g2(static_cast<unsigned>(ceil_div(sd.m, 2 * PEN2_T)), static_cast<unsigned>(ceil_div(P, PH)));
      k_spmm_pencil2<PH, 4><<<g2, PEN2_T, sm2, L.s>>>(static_cast<int>(sd.m), npen, A, x, out, P, sc, pt);
    } else if (sd.W == 4) {
      set_max_dynamic_smem(reinterpret_cast<const void*>(k_spmm_pencil<EF_MAXP, 4>),
                           static_cast<int>(sizeof(double) * EF_MAXP * (PEN_T + 6)));
      k_spmm_pencil<EF_MAXP, 4><<<blocks, PEN_T, smem, L.s>>>(static_cast<int>(sd.m), npen, A, x, out, P, sc, pt);
    } else {
      set_max_dynamic_smem(reinterpret_cast<const void*>(k_spmm_pencil<EF_MAXP, 2>),
                           static_cast<int>(sizeof(double) * EF_MAXP * (PEN_T + 2)));
      k_spmm_pencil<EF_MAXP, 2><<<blocks, PEN_T, smem, L.s>>>(static_cast<int>(sd.m), npen, A, x, out, P, sc, pt);
    }
    return;
  }
  const unsigned blocks = static_cast<unsigned>(ceil_div(sd.m, 128));
  const StencilOffsets off = make_stencil_offsets(sd);
  switch (sd.S_min) {
    case 172: k_spmm<EF_MAXP, 172><<<blocks, 128, 0, L.s>>>(sd.m, A, x, out, P, sc, off); break;
    case 25: k_spmm<EF_MAXP, 25><<<blocks, 128, 0, L.s>>>(sd.m, A, x, out, P, sc, off); break;
    case 4: k_spmm<EF_MAXP, 4><<<blocks, 128, 0, L.s>>>(sd.m, A, x, out, P, sc, off); break;
    case 14: k_spmm<EF_MAXP, 14><<<blocks, 128, 0, L.s>>>(sd.m, A, x, out, P, sc, off); break;
    case 5: k_spmm<EF_MAXP, 5><<<blocks, 128, 0, L.s>>>(sd.m, A, x, out, P, sc, off); break;
    default: k_spmm<EF_MAXP, 2><<<blocks, 128, 0, L.s>>>(sd.m, A, x, out, P, sc, off); break;
  }
}

// s_next += s2·wv ; partials p_next·wv, wv·wt
__global__ void __launch_bounds__(EF_NT) k_ef_s3(int64_t m, double s2, const EfScal* sc, double* snext,
                                                 const double* pnext, const double* wv, const double* wt, double* part,
                                                 int nblk) {
  __shared__ double sh[8];
  const int p = blockIdx.y;
  const bool dn = sc[p].done;
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  double d0 = 0.0, d1 = 0.0;
  if (!dn && a < m) {
    const int64_t o = static_cast<int64_t>(p) * m + a;
    snext[o] += s2 * wv[o];
    d0 = pnext[o] * wv[o];
    d1 = wv[o] * wt[o];
  }
  block_partial_store(d0, part + (static_cast<int64_t>(p) * 2 + 0) * nblk + blockIdx.x, sh);
  block_partial_store(d1, part + (static_cast<int64_t>(p) * 2 + 1) * nblk + blockIdx.x, sh);
}

// β, breakdown (solvers.cpp:513-520)
__global__ void k_ef_c3(int P, int i, int k, EfScal* sc, const double* dots, double* beta, double* dv) {
  const int p = threadIdx.x;
  if (p >= P) return;
  EfScal s = sc[p];
  if (s.done) return;
  const double b = sqrt(fmax(0.0, dots[p * 2 + 0] + 2.0 * s.e * dots[p * 2 + 1] + s.e * s.e));
  if (b <= 1e-12 * fmax(s.scale, 1e-300)) {
    s.done = 1;
    s.order = i + 1;
    sc[p] = s;
    return;
  }
  beta[p * k + i] = b;
  s.scale = fmax(s.scale, b);
  s.b = b;
  s.cqp = s.cq;
  s.cq = s.e / b;
  dv[p * k + i + 1] = s.cq;
  s.bprev = b;
  sc[p] = s;
}

// q_prev = q; q = wv/b; pcur = p_next/b; sbar = s_next/b; store columns; partial q·wt
__global__ void __launch_bounds__(EF_NT) k_ef_s4(int64_t m, int i, int k, const EfScal* sc, double* qprev, double* q,
                                                 const double* wv, double* pcur, const double* pnext, double* sbar,
                                                 const double* snext, double* Qh, double* Ph, const double* wt,
                                                 double* part, int nblk) {
  __shared__ double sh[8];
  const int p = blockIdx.y;
  const EfScal s = sc[p];
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  double d0 = 0.0;
  if (!s.done && a < m) {
    const int64_t o = static_cast<int64_t>(p) * m + a;
    qprev[o] = q[o];
    const double qn = wv[o] / s.b;
    const double pn = pnext[o] / s.b;
    q[o] = qn;
    pcur[o] = pn;
    sbar[o] = snext[o] / s.b;
    Qh[(static_cast<int64_t>(p) * k + i + 1) * m + a] = qn;
    Ph[(static_cast<int64_t>(p) * k + i + 1) * m + a] = pn;
    d0 = qn * wt[o];
  }
  block_partial_store(d0, part + static_cast<int64_t>(p) * nblk + blockIdx.x, sh);
}

__global__ void k_ef_c4(int P, int i, int k, const EfScal* sc, const double* dots, double* tq) {
  const int p = threadIdx.x;
  if (p >= P || sc[p].done) return;
  tq[p * k + i + 1] = dots[p];
}

// normalised start images: wt /= ‖b‖, kwt /= ‖b‖  (solvers.cpp:472-474)
__global__ void k_ef_init(int64_t m, int P, const double* z0sq, const double* wt_in, const double* kwt_in, double* wt,
                          double* kwt) {
  const int p = blockIdx.y;
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  if (a >= m) return;
  const double bn = sqrt(z0sq[p]);
  const int64_t o = static_cast<int64_t>(p) * m + a;
  wt[o] = wt_in[o] / bn;
  kwt[o] = kwt_in[o] / bn;
}

__global__ void k_ef_scal_init(int P, EfScal* sc, double* dv, int k) {
  const int p = threadIdx.x;
  if (p >= P) return;
  EfScal s{};
  s.cq = 1.0;
  sc[p] = s;
  dv[p * k] = 1.0;
}

__global__ void k_add_scaled(int64_t n, double a, const double* x, double* y) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] += a * x[i];
}

// --------------------------------------------------------------- host driver
struct DevMem {
  void* p = nullptr;
  explicit DevMem(size_t bytes) {
    GSGPC_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 64)));
  }
  ~DevMem() {
    if (p) cudaFree(p);
  }
  double* d() const { return static_cast<double*>(p); }
};

void run_kg_batched(const Launch& L, const KgDev& kg, int P, const double* v, double* out, double* t0, double* t1) {
  run_kg_apply_batched(L, kg, P, v, out, t0, t1);
}

// Runs EFLA for P ≤ 32 probes; inputs are device arrays (P × m).
EflaOut efla_run(const Launch& L, const StencilDesc& sd, const double* A, const KgDev& kg, int P, const double* kwt_in,
                 const double* wt_in, const double* z0sq_dev, double s2, int k, double* basis_out) {
  if (P < 1 || P > EF_MAXP) throw Error(GSGPC_UNSUPPORTED, "factorized_lanczos_fused: 1..32 start vectors per batch");
  if (k < 1) invalid("factorized_lanczos_fused: bad k");
  const int64_t m = sd.m;
  const int64_t pm = static_cast<int64_t>(P) * m;
  const int nblk = static_cast<int>(ceil_div(m, EF_NT));
  const size_t V = sizeof(double) * pm;
  DevMem wt(V), kwt(V), q(V), qprev(V), sbar(V), pcur(V), wv(V), pnext(V), snext(V), t0(V), t1(V);
  DevMem Qh(V * k), Ph(V * k);
  DevMem part(sizeof(double) * static_cast<size_t>(P) * (k + 2) * nblk);
  DevMem dots(sizeof(double) * P * (k + 2));
  DevMem lam(sizeof(double) * P * k), tq(sizeof(double) * P * k), dv(sizeof(double) * P * k);
  DevMem al(sizeof(double) * P * k), be(sizeof(double) * P * k);
  DevMem scm(sizeof(EfScal) * P);
  EfScal* sc = static_cast<EfScal*>(scm.p);
  for (DevMem* b : {&q, &qprev, &sbar, &pcur, &Qh, &Ph}) {
    GSGPC_CUDA(cudaMemsetAsync(b->p, 0, b == &Qh || b == &Ph ? V * k : V, L.s));
  }
  for (DevMem* b : {&tq, &dv, &al, &be}) GSGPC_CUDA(cudaMemsetAsync(b->p, 0, sizeof(double) * P * k, L.s));
  const dim3 gv(static_cast<unsigned>(nblk), static_cast<unsigned>(P));
  k_ef_init<<<gv, EF_NT, 0, L.s>>>(m, P, z0sq_dev, wt_in, kwt_in, wt.d(), kwt.d());
  k_ef_scal_init<<<1, 32, 0, L.s>>>(P, sc, dv.d(), k);
  L.count(2);
  for (int i = 0; i < k; ++i) {
    k_ef_s1<<<gv, EF_NT, 0, L.s>>>(m, sc, sbar.d(), kwt.d(), qprev.d(), wv.d(), pcur.d(), wt.d(), part.d(), nblk);
    k_ef_reduce<<<P * 2, EF_NT, 0, L.s>>>(part.d(), nblk, dots.d());
    k_ef_c1<<<1, 32, 0, L.s>>>(P, i, k, s2, sc, dots.d(), tq.d(), al.d());
    L.count(3);
    if (i == k - 1) break;
    k_ef_s2<<<gv, EF_NT, 0, L.s>>>(m, i, k, sc, wv.d(), q.d(), wt.d(), Ph.d(), part.d(), nblk);
    k_ef_reduce<<<P * (i + 2), EF_NT, 0, L.s>>>(part.d(), nblk, dots.d());
    k_ef_c2<<<1, 32, 0, L.s>>>(P, i, k, sc, dots.d(), tq.d(), dv.d(), lam.d());
    k_ef_g2<<<gv, EF_NT, 0, L.s>>>(m, i, k, sc, wv.d(), Qh.d(), lam.d());
    launch_spmm(L, sd, A, wv.d(), pnext.d(), P, sc);
    L.count(5);
    run_kg_batched(L, kg, P, pnext.d(), snext.d(), t0.d(), t1.d());
    k_ef_s3<<<gv, EF_NT, 0, L.s>>>(m, s2, sc, snext.d(), pnext.d(), wv.d(), wt.d(), part.d(), nblk);
    k_ef_reduce<<<P * 2, EF_NT, 0, L.s>>>(part.d(), nblk, dots.d());
    k_ef_c3<<<1, 32, 0, L.s>>>(P, i, k, sc, dots.d(), be.d(), dv.d());
    k_ef_s4<<<gv, EF_NT, 0, L.s>>>(m, i, k, sc, qprev.d(), q.d(), wv.d(), pcur.d(), pnext.d(), sbar.d(), snext.d(),
                                   Qh.d(), Ph.d(), wt.d(), part.d(), nblk);
    k_ef_reduce<<<P, EF_NT, 0, L.s>>>(part.d(), nblk, dots.d());
    k_ef_c4<<<1, 32, 0, L.s>>>(P, i, k, sc, dots.d(), tq.d());
    L.count(6);
  }
  GSGPC_CUDA(cudaGetLastError());
  EflaOut o;
  o.alpha.resize(static_cast<size_t>(P) * k);
  o.beta.resize(static_cast<size_t>(P) * k);
  std::vector<EfScal> hs(P);
  GSGPC_CUDA(cudaMemcpyAsync(o.alpha.data(), al.p, sizeof(double) * P * k, cudaMemcpyDeviceToHost, L.s));
  GSGPC_CUDA(cudaMemcpyAsync(o.beta.data(), be.p, sizeof(double) * P * k, cudaMemcpyDeviceToHost, L.s));
  GSGPC_CUDA(cudaMemcpyAsync(hs.data(), scm.p, sizeof(EfScal) * P, cudaMemcpyDeviceToHost, L.s));
  o.d.resize(static_cast<size_t>(P) * k);
  GSGPC_CUDA(cudaMemcpyAsync(o.d.data(), dv.p, sizeof(double) * P * k, cudaMemcpyDeviceToHost, L.s));
  if (basis_out) GSGPC_CUDA(cudaMemcpyAsync(basis_out, Qh.p, V * k, cudaMemcpyDeviceToDevice, L.s));
  GSGPC_CUDA(cudaStreamSynchronize(L.s));
  o.order.resize(P);
  for (int p = 0; p < P; ++p) o.order[p] = hs[p].order > 0 ? hs[p].order : k;
  return o;
}

// Symmetric tridiagonal eigenproblem (implicit QL, Wilkinson shifts): eigenvalues in
// ascending order and the first component of each eigenvector — what quadrature_logdet
// reads from Eigen's computeFromTridiagonal (gp.cpp:38-56).
void tridiag_eig_host(int n, const double* alpha, const double* beta, std::vector<double>& dd,
                      std::vector<double>& z) {
  dd.assign(alpha, alpha + n);
  std::vector<double> e(n, 0.0);
  for (int i = 0; i + 1 < n; ++i) e[i] = beta[i];
  z.assign(n, 0.0);
  z[0] = 1.0;
  for (int l = 0; l < n; ++l) {
    int iter = 0, mm;
    do {
      for (mm = l; mm < n - 1; ++mm) {
        const double s = std::fabs(dd[mm]) + std::fabs(dd[mm + 1]);
        if (std::fabs(e[mm]) <= 2.220446049250313e-16 * s) break;
      }
      if (mm != l) {
        if (++iter > 200) throw Error(GSGPC_RUNTIME_ERROR, "tridiagonal eigensolver did not converge");
        double g = (dd[l + 1] - dd[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = dd[mm] - dd[l] + e[l] / (g + std::copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        bool early = false;
        for (int i = mm - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = std::hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            dd[i + 1] -= p;
            e[mm] = 0.0;
            early = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = dd[i + 1] - p;
          r = (dd[i] - g) * s + 2.0 * c * b;
          p = s * r;
          dd[i + 1] = g + p;
          g = c * r - b;
          f = z[i + 1];
          z[i + 1] = s * z[i] + c * f;
          z[i] = c * z[i] - s * f;
        }
        if (early) continue;
        dd[l] -= p;
        e[l] = g;
        e[mm] = 0.0;
      }
    } while (mm != l);
  }
  std::vector<int> ord(n);
  for (int i = 0; i < n; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return dd[a] < dd[b]; });
  std::vector<double> d2(n), z2(n);
  for (int i = 0; i < n; ++i) {
    d2[i] = dd[ord[i]];
    z2[i] = z[ord[i]];
  }
  dd.swap(d2);
  z.swap(z2);
}

// quadrature_logdet (gp.cpp:34-63)
std::pair<double, int> quadrature_logdet_host(const double* alpha, const double* beta, int k, double probe_sq,
                                              double quad_tol) {
  double prev = 0.0, value = 0.0;
  int depth = 0;
  std::vector<double> lam, z;
  for (int j = 1; j <= k; ++j) {
    tridiag_eig_host(j, alpha, beta, lam, z);
    double mx = 0.0;
    for (double v : lam) mx = std::max(mx, std::fabs(v));
    const double scale = std::max(mx, 1e-300);
    if (lam[0] < -1e-10 * scale) {
      throw Error(GSGPC_RUNTIME_ERROR, "slq_logdet: negative Ritz value, operator is not positive definite");
    }
    double est = 0.0;
    for (int l = 0; l < j; ++l) est += z[l] * z[l] * std::log(std::max(lam[l], 1e-16 * scale));
    est *= probe_sq;
    value = est;
    depth = j;
    if (j >= 2 && quad_tol > 0.0 && std::fabs(est - prev) <= quad_tol * std::max(std::fabs(est), 1e-300)) break;
    prev = est;
  }
  return {value, depth};
}


// =============================================================== plain Lanczos, batched
// lanczos (solvers.cpp:351-389) for P start vectors at once on an m-dimensional operator:
// classical Gram–Schmidt full reorthogonalisation exactly as the reference orders it
// (w -= β q_{i-1}; α = q·w; w -= α q; c = Qᵀw; w -= Q c; β = ‖w‖; breakdown when
// β ≤ 1e-12·scale).  Used by slq_logdet (gp.cpp:67-83) on the SymmetricGrid route and by
// estimate_grid_kernel_condition (gp.cpp:142-154).
struct LzScal {
  double bprev, scale;
  int done, order;
};

// w -= bprev·q_prev (i > 0); partial q_i·w
__global__ void __launch_bounds__(EF_NT) k_lz_s1(int64_t m, int i, int k, const LzScal* sc, double* w, const double* Q,
                                                 double* part, int nblk) {
  __shared__ double sh[8];
  const int p = blockIdx.y;
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  const bool live = !sc[p].done && a < m;
  double v = 0.0;
  if (live) {
    const int64_t o = static_cast<int64_t>(p) * m + a;
    const double* Qp = Q + static_cast<int64_t>(p) * k * m;
    double x = w[o];
    if (i > 0) x -= sc[p].bprev * Qp[static_cast<int64_t>(i - 1) * m + a];
    w[o] = x;
    v = Qp[static_cast<int64_t>(i) * m + a] * x;
  }
  block_partial_store(v, part + static_cast<int64_t>(p) * nblk + blockIdx.x, sh);
}

__global__ void k_lz_c1(int P, int i, int k, LzScal* sc, const double* dots, double* alpha) {
  const int p = threadIdx.x;
  if (p >= P || sc[p].done) return;
  const double a = dots[p];
  alpha[p * k + i] = a;
  sc[p].scale = fmax(sc[p].scale, fabs(a));
  if (i == k - 1) {
    sc[p].done = 1;
    sc[p].order = k;
  }
}

// w -= α q_i; partials q_j·w (j ≤ i)
__global__ void __launch_bounds__(EF_NT) k_lz_s2(int64_t m, int i, int k, const LzScal* sc, const double* alpha,
                                                 double* w, const double* Q, double* part, int nblk) {
  __shared__ double sh[8];
  const int p = blockIdx.y;
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  const bool live = !sc[p].done && a < m;
  const double* Qp = Q + static_cast<int64_t>(p) * k * m;
  double x = 0.0;
  if (live) {
    const int64_t o = static_cast<int64_t>(p) * m + a;
    x = w[o] - alpha[p * k + i] * Qp[static_cast<int64_t>(i) * m + a];
    w[o] = x;
  }
  for (int j = 0; j <= i; ++j) {
    const double v = live ? Qp[static_cast<int64_t>(j) * m + a] * x : 0.0;
    block_partial_store(v, part + (static_cast<int64_t>(p) * (i + 1) + j) * nblk + blockIdx.x, sh);
  }
}

// w -= Σ_j q_j c_j; partial w·w
__global__ void __launch_bounds__(EF_NT) k_lz_g2(int64_t m, int i, int k, const LzScal* sc, const double* c, double* w,
                                                 const double* Q, double* part, int nblk) {
  __shared__ double sh[8];
  const int p = blockIdx.y;
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  const bool live = !sc[p].done && a < m;
  double v = 0.0;
  if (live) {
    const double* Qp = Q + static_cast<int64_t>(p) * k * m;
    const int64_t o = static_cast<int64_t>(p) * m + a;
    double x = w[o];
    for (int j = 0; j <= i; ++j) x -= Qp[static_cast<int64_t>(j) * m + a] * c[p * (i + 1) + j];
    w[o] = x;
    v = x * x;
  }
  block_partial_store(v, part + static_cast<int64_t>(p) * nblk + blockIdx.x, sh);
}

__global__ void k_lz_c3(int P, int i, int k, LzScal* sc, const double* dots, double* beta) {
  const int p = threadIdx.x;
  if (p >= P || sc[p].done) return;
  const double b = sqrt(dots[p]);
  if (b <= 1e-12 * fmax(sc[p].scale, 1e-300)) {
    sc[p].done = 1;
    sc[p].order = i + 1;
    return;
  }
  beta[p * k + i] = b;
  sc[p].scale = fmax(sc[p].scale, b);
  sc[p].bprev = b;
}

// q_{i+1} = w / β (into Q and the contiguous operator input)
__global__ void __launch_bounds__(EF_NT) k_lz_s4(int64_t m, int i, int k, const LzScal* sc, const double* w, double* Q,
                                                 double* cur) {
  const int p = blockIdx.y;
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  if (sc[p].done || a >= m) return;
  const int64_t o = static_cast<int64_t>(p) * m + a;
  const double q = w[o] / sc[p].bprev;
  Q[(static_cast<int64_t>(p) * k + i + 1) * m + a] = q;
  cur[o] = q;
}

// q_0 = b / ‖b‖ (‖b‖ from a device reduction)
__global__ void __launch_bounds__(EF_NT) k_lz_init(int64_t m, int k, const double* b, const double* bb, double* Q,
                                                   double* cur) {
  const int p = blockIdx.y;
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  if (a >= m) return;
  const int64_t o = static_cast<int64_t>(p) * m + a;
  const double q = b[o] / sqrt(bb[p]);
  Q[static_cast<int64_t>(p) * k * m + a] = q;
  cur[o] = q;
}

__global__ void __launch_bounds__(EF_NT) k_lz_sq(int64_t m, const double* b, double* part, int nblk) {
  __shared__ double sh[8];
  const int p = blockIdx.y;
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  const double v = a < m ? b[static_cast<int64_t>(p) * m + a] : 0.0;
  block_partial_store(v * v, part + static_cast<int64_t>(p) * nblk + blockIdx.x, sh);
}

__global__ void k_lz_scal_init(int P, LzScal* sc) {
  const int p = threadIdx.x;
  if (p < P) sc[p] = LzScal{0.0, 0.0, 0, 0};
}

// out = op(in) for P probe-major vectors
using BatchedOp = std::function<void(const double* in, double* out)>;

LanczosOut lanczos_batched(const Launch& L, int64_t m, int P, int k, const double* start, const BatchedOp& op) {
  if (k < 1 || k > m) invalid("lanczos: need 1 <= k <= dim");
  const int nblk = static_cast<int>(ceil_div(m, EF_NT));
  const size_t V = sizeof(double) * static_cast<size_t>(P) * m;
  DevMem Q(V * k), cur(V), w(V);
  DevMem part(sizeof(double) * static_cast<size_t>(P) * (k + 1) * nblk), dots(sizeof(double) * P * (k + 1));
  DevMem al(sizeof(double) * P * k), be(sizeof(double) * P * k), scm(sizeof(LzScal) * P);
  LzScal* sc = static_cast<LzScal*>(scm.p);
  GSGPC_CUDA(cudaMemsetAsync(al.p, 0, sizeof(double) * P * k, L.s));
  GSGPC_CUDA(cudaMemsetAsync(be.p, 0, sizeof(double) * P * k, L.s));
  const dim3 gv(static_cast<unsigned>(nblk), static_cast<unsigned>(P));
  k_lz_sq<<<gv, EF_NT, 0, L.s>>>(m, start, part.d(), nblk);
  k_ef_reduce<<<P, EF_NT, 0, L.s>>>(part.d(), nblk, dots.d());
  std::vector<double> bb(P);
  GSGPC_CUDA(cudaMemcpyAsync(bb.data(), dots.p, sizeof(double) * P, cudaMemcpyDeviceToHost, L.s));
  GSGPC_CUDA(cudaStreamSynchronize(L.s));
  for (double v : bb)
    if (v == 0.0) invalid("lanczos: start vector is zero");
  k_lz_init<<<gv, EF_NT, 0, L.s>>>(m, k, start, dots.d(), Q.d(), cur.d());
  k_lz_scal_init<<<1, 64, 0, L.s>>>(P, sc);
  L.count(4);
  for (int i = 0; i < k; ++i) {
    op(cur.d(), w.d());
    k_lz_s1<<<gv, EF_NT, 0, L.s>>>(m, i, k, sc, w.d(), Q.d(), part.d(), nblk);
    k_ef_reduce<<<P, EF_NT, 0, L.s>>>(part.d(), nblk, dots.d());
    k_lz_c1<<<1, 64, 0, L.s>>>(P, i, k, sc, dots.d(), al.d());
    L.count(3);
    if (i == k - 1) break;
    k_lz_s2<<<gv, EF_NT, 0, L.s>>>(m, i, k, sc, al.d(), w.d(), Q.d(), part.d(), nblk);
    k_ef_reduce<<<P * (i + 1), EF_NT, 0, L.s>>>(part.d(), nblk, dots.d());
    k_lz_g2<<<gv, EF_NT, 0, L.s>>>(m, i, k, sc, dots.d(), w.d(), Q.d(), part.d(), nblk);
    k_ef_reduce<<<P, EF_NT, 0, L.s>>>(part.d(), nblk, dots.d());
    k_lz_c3<<<1, 64, 0, L.s>>>(P, i, k, sc, dots.d(), be.d());
    k_lz_s4<<<gv, EF_NT, 0, L.s>>>(m, i, k, sc, w.d(), Q.d(), cur.d());
    L.count(6);
  }
  GSGPC_CUDA(cudaGetLastError());
  LanczosOut o;
  o.alpha.resize(static_cast<size_t>(P) * k);
  o.beta.resize(static_cast<size_t>(P) * k);
  std::vector<LzScal> hs(P);
  GSGPC_CUDA(cudaMemcpyAsync(o.alpha.data(), al.p, sizeof(double) * P * k, cudaMemcpyDeviceToHost, L.s));
  GSGPC_CUDA(cudaMemcpyAsync(o.beta.data(), be.p, sizeof(double) * P * k, cudaMemcpyDeviceToHost, L.s));
  GSGPC_CUDA(cudaMemcpyAsync(hs.data(), scm.p, sizeof(LzScal) * P, cudaMemcpyDeviceToHost, L.s));
  GSGPC_CUDA(cudaStreamSynchronize(L.s));
  o.order.resize(P);
  for (int p = 0; p < P; ++p) o.order[p] = hs[p].order > 0 ? hs[p].order : k;
  return o;
}

// rademacher_probe (gp.cpp:16-25) for p0 .. p0+P-1, dimension m, probe-major ±1 doubles
static std::vector<double> rademacher_block(int64_t m, uint64_t seed, int p0, int P) {
  std::vector<double> v(static_cast<size_t>(P) * m);
  for (int p = 0; p < P; ++p) {
    const uint64_t pi = static_cast<uint64_t>(p0 + p);
    std::seed_seq seq{static_cast<std::uint32_t>(seed), static_cast<std::uint32_t>(seed >> 32),
                      static_cast<std::uint32_t>(pi), static_cast<std::uint32_t>(pi >> 32)};
    std::mt19937_64 rng(seq);
    double* o = v.data() + static_cast<size_t>(p) * m;
    for (int64_t i = 0; i < m; ++i) o[i] = (rng() & 1ull) ? 1.0 : -1.0;
  }
  return v;
}

// slq_logdet (gp.cpp:67-83) with the probes batched EF_MAXP at a time
// Σ of the per-probe quadrature estimates over probes [p_begin, p_end) (the caller divides by
// the total probe count: shards of the probe set add up across ranks)
double slq_logdet_sum(const Launch& L, int64_t m, int p_begin, int p_end, int max_depth, double quad_tol,
                      uint64_t seed, const std::function<BatchedOp(int)>& make_op) {
  const int depth = static_cast<int>(std::min<int64_t>(max_depth, m));
  double total = 0.0;
  for (int p0 = p_begin; p0 < p_end; p0 += EF_MAXP) {
    const int P = std::min(EF_MAXP, p_end - p0);
    const std::vector<double> hv = rademacher_block(m, seed, p0, P);
    DevMem dv(sizeof(double) * hv.size());
    GSGPC_CUDA(cudaMemcpyAsync(dv.p, hv.data(), sizeof(double) * hv.size(), cudaMemcpyHostToDevice, L.s));
    const LanczosOut o = lanczos_batched(L, m, P, depth, dv.d(), make_op(P));
    for (int p = 0; p < P; ++p) {
      total += quadrature_logdet_host(o.alpha.data() + static_cast<size_t>(p) * depth,
                                      o.beta.data() + static_cast<size_t>(p) * depth, o.order[p],
                                      static_cast<double>(m), quad_tol)
                   .first;
    }
  }
  return total;
}

// Batched operators of the SymmetricGrid route
BatchedOp kg_op(const Launch& L, const KgDev& kg, int P, double* t0, double* t1) {
  return [=](const double* in, double* out) { run_kg_batched(L, kg, P, in, out, t0, t1); };
}

// out = K WᵀW K u + σ² K u
BatchedOp sym_op(const Launch& L, const StencilDesc& sd, const double* A, const KgDev& kg, int P, double sigma_sq,
                 double* ku, double* wku, double* t0, double* t1) {
  return [=](const double* in, double* out) {
    run_kg_batched(L, kg, P, in, ku, t0, t1);
    launch_spmm(L, sd, A, ku, wku, P, nullptr);
    run_kg_batched(L, kg, P, wku, out, t0, t1);
    const int64_t n = static_cast<int64_t>(P) * sd.m;
    k_add_scaled<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, L.s>>>(n, sigma_sq, ku, out);
    L.count(2);
  };
}

// estimate_grid_kernel_condition (gp.cpp:142-154): Lanczos on K_G from probe 0 of seed
// 0x5eedf00d, depth min(30, m); hi / max(lo, 1e-18·hi) of the Ritz values.
double kg_condition_estimate(const Launch& L, const KgDev& kg) {
  const int64_t m = kg.m;
  const int depth = static_cast<int>(std::min<int64_t>(30, m));
  const std::vector<double> hv = rademacher_block(m, 0x5eedf00dull, 0, 1);
  DevMem dv(sizeof(double) * m), t0(sizeof(double) * m), t1(sizeof(double) * m);
  GSGPC_CUDA(cudaMemcpyAsync(dv.p, hv.data(), sizeof(double) * m, cudaMemcpyHostToDevice, L.s));
  const LanczosOut o = lanczos_batched(L, m, 1, depth, dv.d(), kg_op(L, kg, 1, t0.d(), t1.d()));
  std::vector<double> lam, z;
  tridiag_eig_host(o.order[0], o.alpha.data(), o.beta.data(), lam, z);
  const double hi = lam.back(), lo = lam.front();
  if (!(hi > 0.0)) return INFINITY;
  return hi / std::max(lo, hi * 1e-18);
}

// ------------------------------------------------------------ Dense route (gp.cpp:116-140)
// log|det(K_G WᵀW + σ² I)| for m ≤ dense_cap: dense K_G (Kronecker of the generators) and
// dense WᵀW (from the half stencil), one DGEMM, then LU with partial pivoting in a single
// cooperative kernel (same pivot rule as the reference: first row of maximal |a|).
__global__ void k_dense_kg(int64_t m, KgDev kg, double* K) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= m * m) return;
  int64_t i = idx / m, j = idx % m;
  double v = 1.0;
  for (int k = kg.d - 1; k >= 0; --k) {
    const int64_t ik = i % kg.sz[k], jk = j % kg.sz[k];
    i /= kg.sz[k];
    j /= kg.sz[k];
    v *= kg.gen[k][ik > jk ? ik - jk : jk - ik];
  }
  K[idx] = v;
}

// dense WᵀW from the half stencil: row a, offset s ≥ 0: (a, a+o_s) and (a+o_s, a)
__global__ void k_dense_wtw(int64_t m, int S_min, const double* A, double* D,
                            const __grid_constant__ StencilOffsets off) {
  const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= m) return;
  for (int s2 = 0; s2 < S_min; ++s2) {
    const int64_t b = a + off.flat[s2];
    if (b < 0 || b >= m) continue;
    const double v = A[static_cast<int64_t>(s2) * m + a];
    if (v == 0.0) continue;
    D[a * m + b] = v;
    D[b * m + a] = v;
  }
}

// C = A·B + σ² I (row-major m×m), 32×32 tiles
__global__ void __launch_bounds__(256) k_dgemm_shift(int m, const double* __restrict__ A, const double* __restrict__ B,
                                                     double sigma_sq, double* __restrict__ C) {
  __shared__ double As[32][33], Bs[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 × 8
  const int row0 = blockIdx.y * 32, col = blockIdx.x * 32 + tx;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k0 = 0; k0 < m; k0 += 32) {
    for (int r = ty; r < 32; r += 8) {
      const int gr = row0 + r, gk = k0 + tx;
      As[r][tx] = (gr < m && gk < m) ? A[static_cast<int64_t>(gr) * m + gk] : 0.0;
      const int bk = k0 + r;
      Bs[r][tx] = (bk < m && col < m) ? B[static_cast<int64_t>(bk) * m + col] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      const double b = Bs[kk][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(As[ty + 8 * q][kk], b, acc[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = row0 + ty + 8 * q;
    if (r < m && col < m) C[static_cast<int64_t>(r) * m + col] = acc[q] + (r == col ? sigma_sq : 0.0);
  }
}

// Right-looking LU with partial pivoting, one cooperative grid; logdet = Σ log|u_cc|.
// Element updates are a[r][j] − f·a[c][j] with f = a[r][c] / a[c][c], rounded as the
// reference's (no contraction).
__global__ void __launch_bounds__(256) k_dense_lu_logdet(int m, double* a, double* red_v, int* red_i, double* out) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sv[256];
  __shared__ int si[256];
  const int nthreads = gridDim.x * blockDim.x;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  double logdet = 0.0;
  for (int c = 0; c < m; ++c) {
    // pivot: first row r ≥ c with maximal |a[r][c]|
    double bv = -1.0;
    int bi = m;
    for (int r = c + tid; r < m; r += nthreads) {
      const double v = fabs(a[static_cast<int64_t>(r) * m + c]);
      if (v > bv || (v == bv && r < bi)) {
        bv = v;
        bi = r;
      }
    }
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if (threadIdx.x < o) {
        const double v2 = sv[threadIdx.x + o];
        const int i2 = si[threadIdx.x + o];
        if (v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 < si[threadIdx.x])) {
          sv[threadIdx.x] = v2;
          si[threadIdx.x] = i2;
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      red_v[blockIdx.x] = sv[0];
      red_i[blockIdx.x] = si[0];
    }
    grid.sync();
    // every thread reduces the block winners identically
    double pv = -1.0;
    int piv = m;
    for (int b = 0; b < static_cast<int>(gridDim.x); ++b) {
      const double v2 = red_v[b];
      const int i2 = red_i[b];
      if (v2 > pv || (v2 == pv && i2 < piv)) {
        pv = v2;
        piv = i2;
      }
    }
    if (piv != c) {
      for (int j = c + tid; j < m; j += nthreads) {
        const double t = a[static_cast<int64_t>(c) * m + j];
        a[static_cast<int64_t>(c) * m + j] = a[static_cast<int64_t>(piv) * m + j];
        a[static_cast<int64_t>(piv) * m + j] = t;
      }
    }
    grid.sync();
    const double dg = a[static_cast<int64_t>(c) * m + c];
    logdet += log(fabs(dg));
    if (dg != 0.0) {
      const int64_t rows = m - c - 1, cols = m - c - 1;
      for (int64_t e = tid; e < rows * cols; e += nthreads) {
        const int r = c + 1 + static_cast<int>(e / cols);
        const int j = c + 1 + static_cast<int>(e % cols);
        const double f = __ddiv_rn(a[static_cast<int64_t>(r) * m + c], dg);
        if (f == 0.0) continue;
        a[static_cast<int64_t>(r) * m + j] =
            __dsub_rn(a[static_cast<int64_t>(r) * m + j], __dmul_rn(f, a[static_cast<int64_t>(c) * m + j]));
      }
    }
    grid.sync();
  }
  if (tid == 0) *out = logdet;
}

double dense_logdet_grid_system(const Launch& L, const StencilDesc& sd, const double* A, const KgDev& kg,
                                double sigma_sq) {
  const int64_t m = sd.m;
  const size_t MM = sizeof(double) * static_cast<size_t>(m) * m;
  DevMem K(MM), D(MM), S(MM);
  GSGPC_CUDA(cudaMemsetAsync(D.p, 0, MM, L.s));
  k_dense_kg<<<static_cast<unsigned>(ceil_div(m * m, 256)), 256, 0, L.s>>>(m, kg, K.d());
  k_dense_wtw<<<static_cast<unsigned>(ceil_div(m, 256)), 256, 0, L.s>>>(m, sd.S_min, A, D.d(),
                                                                      make_stencil_offsets(sd));
  const dim3 gg(static_cast<unsigned>(ceil_div(m, 32)), static_cast<unsigned>(ceil_div(m, 32)));
  k_dgemm_shift<<<gg, 256, 0, L.s>>>(static_cast<int>(m), K.d(), D.d(), sigma_sq, S.d());
  L.count(3);
  int dev = 0, sms = 0, per_sm = 0;
  GSGPC_CUDA(cudaGetDevice(&dev));
  GSGPC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  GSGPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dense_lu_logdet, 256, 0));
  const int blocks = std::max(1, sms * std::min(per_sm, 2));
  DevMem rv(sizeof(double) * blocks), ri(sizeof(int) * blocks), out(sizeof(double));
  int mi = static_cast<int>(m);
  double* ap = S.d();
  double* rvp = rv.d();
  int* rip = static_cast<int*>(ri.p);
  double* op = out.d();
  void* args[] = {&mi, &ap, &rvp, &rip, &op};
  GSGPC_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_dense_lu_logdet), dim3(blocks), dim3(256), args, 0,
                                         L.s));
  L.count();
  double h = 0.0;
  GSGPC_CUDA(cudaMemcpyAsync(&h, out.p, sizeof(double), cudaMemcpyDeviceToHost, L.s));
  GSGPC_CUDA(cudaStreamSynchronize(L.s));
  return h;
}


// =============================================================== multi-RHS EFCG
// factorized_cg_grid_rhs (solvers.cpp:271-336) for P right-hand sides at once: one stencil
// read per iteration serves every RHS (k_spmm), K_G runs batched, per-RHS scalars (ρ, eps,
// α, β, iterations, done/converged/breakdown) live on the device; each RHS follows exactly
// its single-RHS recurrence and freezes when it converges.
struct BcgScal {
  double rho, eps, alpha, beta;
  int iters, done, converged, breakdown;
};

// partial dots x_p · y_p
__global__ void __launch_bounds__(EF_NT) k_bcg_dot(int64_t m, const double* x, const double* y, double* part,
                                                   int nblk) {
  __shared__ double sh[8];
  const int p = blockIdx.y;
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  const double v = a < m ? x[static_cast<int64_t>(p) * m + a] * y[static_cast<int64_t>(p) * m + a] : 0.0;
  block_partial_store(v, part + static_cast<int64_t>(p) * nblk + blockIdx.x, sh);
}

// v += σ² r; s = u; z = v (init)
__global__ void __launch_bounds__(EF_NT) k_bcg_init_dir(int64_t n, double s2, const double* r, const double* u, double* v,
                                                        double* sdir, double* z) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  if (i >= n) return;
  const double vv = v[i] + s2 * r[i];
  v[i] = vv;
  sdir[i] = u[i];
  z[i] = vv;
}

__global__ void k_bcg_c0(int P, double eps_abs, double rel_tol, BcgScal* sc, const double* dots) {
  const int p = threadIdx.x;
  if (p >= P) return;
  BcgScal s{};
  s.rho = dots[p];
  s.eps = eps_abs >= 0.0 ? eps_abs : rel_tol * rel_tol * s.rho;
  if (s.rho <= s.eps) {
    s.done = 1;
    s.converged = 1;
  }
  sc[p] = s;
}

// pap → α (breakdown when pap ≤ 0)
__global__ void k_bcg_c1(int P, int maxiter, BcgScal* sc, const double* dots) {
  const int p = threadIdx.x;
  if (p >= P) return;
  BcgScal s = sc[p];
  if (s.done) return;
  if (s.iters >= maxiter) {
    s.done = 1;
  } else if (!(dots[p] > 0.0)) {
    s.breakdown = 1;
    s.done = 1;
  } else {
    s.alpha = s.rho / dots[p];
  }
  sc[p] = s;
}

// x += α s; r −= α z
__global__ void __launch_bounds__(EF_NT) k_bcg_upd(int64_t m, const BcgScal* sc, double* x, double* r, const double* sdir,
                                                   const double* z) {
  const int p = blockIdx.y;
  if (sc[p].done) return;
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  if (a >= m) return;
  const int64_t o = static_cast<int64_t>(p) * m + a;
  const double al = sc[p].alpha;
  x[o] += al * sdir[o];
  r[o] -= al * z[o];
}

// v += σ² r (live RHS); partial u·r
__global__ void __launch_bounds__(EF_NT) k_bcg_v(int64_t m, double s2, const BcgScal* sc, const double* r,
                                                 const double* u, double* v, double* part, int nblk) {
  __shared__ double sh[8];
  const int p = blockIdx.y;
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  double d = 0.0;
  if (!sc[p].done && a < m) {
    const int64_t o = static_cast<int64_t>(p) * m + a;
    v[o] += s2 * r[o];
    d = u[o] * r[o];
  }
  block_partial_store(d, part + static_cast<int64_t>(p) * nblk + blockIdx.x, sh);
}

// ρ' → converged / β
__global__ void k_bcg_c2(int P, BcgScal* sc, const double* dots) {
  const int p = threadIdx.x;
  if (p >= P) return;
  BcgScal s = sc[p];
  if (s.done) return;
  const double rn = dots[p];
  s.iters += 1;
  if (rn <= s.eps) {
    s.converged = 1;
    s.done = 1;
    s.rho = rn;
    s.beta = 0.0;
  } else {
    s.beta = rn / s.rho;
    s.rho = rn;
  }
  sc[p] = s;
}

// s = u + β s; z = v + β z (RHS still iterating)
__global__ void __launch_bounds__(EF_NT) k_bcg_dir(int64_t m, const BcgScal* sc, const double* u, const double* v,
                                                   double* sdir, double* z) {
  const int p = blockIdx.y;
  if (sc[p].done) return;
  const int64_t a = static_cast<int64_t>(blockIdx.x) * EF_NT + threadIdx.x;
  if (a >= m) return;
  const int64_t o = static_cast<int64_t>(p) * m + a;
  const double b = sc[p].beta;
  sdir[o] = u[o] + b * sdir[o];
  z[o] = v[o] + b * z[o];
}

BcgOut bcg_run(const Launch& L, const StencilDesc& sd, const double* A, const KgDev& kg, int P, const double* rhat0,
               double sigma, double eps_abs, double rel_tol, int maxiter, double* x) {
  if (P < 1 || P > EF_MAXP) throw Error(GSGPC_UNSUPPORTED, "multi-RHS EFCG: 1..32 right-hand sides per batch");
  const int64_t m = sd.m;
  const int64_t pm = static_cast<int64_t>(P) * m;
  const int nblk = static_cast<int>(ceil_div(m, EF_NT));
  const size_t V = sizeof(double) * pm;
  const double s2 = sigma * sigma;
  DevMem r(V), u(V), v(V), sdir(V), z(V), t0(V), t1(V);
  DevMem part(sizeof(double) * P * nblk), dots(sizeof(double) * P), scm(sizeof(BcgScal) * P);
  BcgScal* sc = static_cast<BcgScal*>(scm.p);
  const dim3 gv(static_cast<unsigned>(nblk), static_cast<unsigned>(P));
  const unsigned gl = static_cast<unsigned>(ceil_div(pm, EF_NT));
  GSGPC_CUDA(cudaMemcpyAsync(r.p, rhat0, V, cudaMemcpyDeviceToDevice, L.s));
  GSGPC_CUDA(cudaMemsetAsync(x, 0, V, L.s));
  launch_spmm(L, sd, A, r.d(), u.d(), P, nullptr);
  run_kg_batched(L, kg, P, u.d(), v.d(), t0.d(), t1.d());
  k_bcg_init_dir<<<gl, EF_NT, 0, L.s>>>(pm, s2, r.d(), u.d(), v.d(), sdir.d(), z.d());
  k_bcg_dot<<<gv, EF_NT, 0, L.s>>>(m, u.d(), r.d(), part.d(), nblk);
  k_ef_reduce<<<P, EF_NT, 0, L.s>>>(part.d(), nblk, dots.d());
  k_bcg_c0<<<1, 64, 0, L.s>>>(P, eps_abs, rel_tol, sc, dots.d());
  L.count(6);
  std::vector<BcgScal> hs(P);
  for (int it = 0; it < maxiter; ++it) {
    k_bcg_dot<<<gv, EF_NT, 0, L.s>>>(m, sdir.d(), z.d(), part.d(), nblk);
    k_ef_reduce<<<P, EF_NT, 0, L.s>>>(part.d(), nblk, dots.d());
    k_bcg_c1<<<1, 64, 0, L.s>>>(P, maxiter, sc, dots.d());
    k_bcg_upd<<<gv, EF_NT, 0, L.s>>>(m, sc, x, r.d(), sdir.d(), z.d());
    launch_spmm(L, sd, A, r.d(), u.d(), P, nullptr);
    run_kg_batched(L, kg, P, u.d(), v.d(), t0.d(), t1.d());
    k_bcg_v<<<gv, EF_NT, 0, L.s>>>(m, s2, sc, r.d(), u.d(), v.d(), part.d(), nblk);
    k_ef_reduce<<<P, EF_NT, 0, L.s>>>(part.d(), nblk, dots.d());
    k_bcg_c2<<<1, 64, 0, L.s>>>(P, sc, dots.d());
    k_bcg_dir<<<gv, EF_NT, 0, L.s>>>(m, sc, u.d(), v.d(), sdir.d(), z.d());
    L.count(9);
    if ((it & 7) == 7 || it + 1 == maxiter) {
      GSGPC_CUDA(cudaMemcpyAsync(hs.data(), scm.p, sizeof(BcgScal) * P, cudaMemcpyDeviceToHost, L.s));
      GSGPC_CUDA(cudaStreamSynchronize(L.s));
      bool all = true;
      for (const auto& q : hs) all = all && q.done;
      if (all) break;
    }
  }
  GSGPC_CUDA(cudaMemcpyAsync(hs.data(), scm.p, sizeof(BcgScal) * P, cudaMemcpyDeviceToHost, L.s));
  GSGPC_CUDA(cudaStreamSynchronize(L.s));
  BcgOut o;
  for (const auto& q : hs) {
    o.iterations.push_back(q.iters);
    o.converged.push_back(q.converged);
    o.breakdown = o.breakdown || q.breakdown;
    o.residual_sq.push_back(q.rho);
  }
  return o;
}

// =============================================================== covariance helpers
// dense W_x rows [ns][m] from compact interp weights (idx/w [ns][cap], nnz)
__global__ void k_cov_scatter_w(int64_t ns, int64_t m, int cap, const int64_t* idx, const double* w, const int* nnz,
                                double* out) {
  const int64_t i = blockIdx.x;
  for (int a = threadIdx.x; a < nnz[i]; a += blockDim.x) out[i * m + idx[i * cap + a]] = w[i * cap + a];
}

// out[i][j] = Σ_a w_i[a] · H[j][idx_i[a]]   (rows of H: nh)
__global__ void k_cov_gather(int64_t ni, int64_t nh, int64_t m, int cap, const int64_t* idx, const double* w,
                             const int* nnz, const double* H, double* out) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ni * nh) return;
  const int64_t i = e / nh, j = e % nh;
  double acc = 0.0;
  for (int a = 0; a < nnz[i]; ++a) acc += w[i * cap + a] * H[j * m + idx[i * cap + a]];
  out[e] = acc;
}

// C[i][j] −= Σ_r A[i][r] B[j][r]   (row-major, 32×32 tiles)
__global__ void __launch_bounds__(256) k_cov_sub_abt(int n, int64_t m, const double* __restrict__ A,
                                                     const double* __restrict__ B, double* __restrict__ C) {
  __shared__ double As[32][33], Bs[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t r0 = 0; r0 < m; r0 += 32) {
    for (int q = ty; q < 32; q += 8) {
      const int64_t rr = r0 + tx;
      As[q][tx] = (i0 + q < n && rr < m) ? A[static_cast<int64_t>(i0 + q) * m + rr] : 0.0;
      Bs[q][tx] = (j0 + q < n && rr < m) ? B[static_cast<int64_t>(j0 + q) * m + rr] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      const double b = Bs[tx][kk];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(As[ty + 8 * q][kk], b, acc[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = i0 + ty + 8 * q, j = j0 + tx;
    if (i < n && j < n) C[static_cast<int64_t>(i) * n + j] -= acc[q];
  }
}

void cov_scatter_w(const Launch& L, int64_t ns, int64_t m, int cap, const int64_t* idx, const double* w,
                   const int* nnz, double* out) {
  GSGPC_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * ns * m, L.s));
  if (ns > 0) k_cov_scatter_w<<<static_cast<unsigned>(ns), 64, 0, L.s>>>(ns, m, cap, idx, w, nnz, out);
  L.count();
}

void cov_gather(const Launch& L, int64_t ni, int64_t nh, int64_t m, int cap, const int64_t* idx, const double* w,
                const int* nnz, const double* H, double* out) {
  if (ni * nh == 0) return;
  k_cov_gather<<<static_cast<unsigned>(ceil_div(ni * nh, 256)), 256, 0, L.s>>>(ni, nh, m, cap, idx, w, nnz, H, out);
  L.count();
}

void cov_sub_abt(const Launch& L, int n, int64_t m, const double* A, const double* B, double* C) {
  if (n == 0) return;
  const dim3 g(static_cast<unsigned>(ceil_div(n, 32)), static_cast<unsigned>(ceil_div(n, 32)));
  k_cov_sub_abt<<<g, 256, 0, L.s>>>(n, m, A, B, C);
  L.count();
}

void spmm_batched(const Launch& L, const StencilDesc& sd, const double* A, const double* x, double* out, int P) {
  for (int p0 = 0; p0 < P; p0 += EF_MAXP) {
    const int pb = std::min(EF_MAXP, P - p0);
    launch_spmm(L, sd, A, x + static_cast<int64_t>(p0) * sd.m, out + static_cast<int64_t>(p0) * sd.m, pb, nullptr);
  }
  L.count();
}

}  // namespace gsgpc
