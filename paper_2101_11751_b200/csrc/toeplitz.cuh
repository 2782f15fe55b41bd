// toeplitz.cuh — one Toeplitz mode product tile (K_G = ⊗_k T_k, T_k symmetric Toeplitz with
// generator g_k[|i-j|]), shared by the standalone mode kernel (operators.cu) and the
// persistent EFCG kernel (efcg_persistent.cu).
//
// Shared memory holds the mirrored generator Ts[1 + q] = g[|q - (n-1)|], q ∈ [0, 2n-2]
// (zero-padded: Ts[0] and Ts[2n .. 2n+3], TOEP_TS(n) doubles) followed by the tile's input
// lines Xs[j][tl] (n × TL).  Each
// thread produces RB = 4 consecutive outputs a..a+3 of one line, so every Xs value is
// loaded once per 4 FMAs and the generator slides through registers (1 new value per j):
// the loop moves 2 shared loads per 4 FMAs instead of 2 per FMA.
#pragma once

#include "internal.cuh"

namespace gsgpc {

constexpr int TOEP_RB = 4;

__host__ __device__ inline int64_t toep_ts_doubles(int64_t n) { return 2 * n + 4; }

// Loads Ts and the X tile; l0 = first line, nl = lines in the tile.
__device__ __forceinline__ void toep_load_tile(const double* __restrict__ X, const double* __restrict__ gen, int64_t n,
                                               int64_t inner, int TL, int64_t l0, int nl, double* Ts, double* Xs,
                                               int nthreads) {
  if (threadIdx.x < 5) Ts[threadIdx.x == 0 ? 0 : 2 * n - 1 + threadIdx.x] = 0.0;
  for (int64_t q = threadIdx.x; q < 2 * n - 1; q += nthreads) {
    const int64_t dd = q - (n - 1);
    Ts[1 + q] = gen[dd < 0 ? -dd : dd];
  }
  // U loads in flight per thread: the tile is ~TL·n doubles from L2 and a one-load-per-
  // iteration loop serialised on its latency
  constexpr int U = 8;
  if (inner == 1) {
    const int64_t cnt = static_cast<int64_t>(nl) * n;
    for (int64_t q0 = threadIdx.x; q0 < cnt; q0 += static_cast<int64_t>(U) * nthreads) {
      double t[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = q0 + static_cast<int64_t>(u) * nthreads;
        t[u] = q < cnt ? __ldcg(X + l0 * n + q) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = q0 + static_cast<int64_t>(u) * nthreads;
        if (q < cnt) Xs[(q % n) * TL + q / n] = t[u];
      }
    }
  } else {
    const int64_t cnt = static_cast<int64_t>(TL) * n;
    for (int64_t q0 = threadIdx.x; q0 < cnt; q0 += static_cast<int64_t>(U) * nthreads) {
      double t[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = q0 + static_cast<int64_t>(u) * nthreads;
        const int tl = static_cast<int>(q % TL);
        const int64_t j = q / TL;
        const int64_t l = l0 + tl, o = l / inner, i = l % inner;
        t[u] = (q < cnt && tl < nl) ? __ldcg(X + (o * n + j) * inner + i) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = q0 + static_cast<int64_t>(u) * nthreads;
        if (q < cnt && static_cast<int>(q % TL) < nl) Xs[(q / TL) * TL + q % TL] = t[u];
      }
    }
  }
}

// Output group u of the tile → (tl, first output a). Groups: nl lines × ceil(na/RB).
__device__ __forceinline__ void toep_group(int uu, int nl, int na, bool inner1, int& tl, int& ar) {
  const int ng = (na + TOEP_RB - 1) / TOEP_RB;
  if (inner1) {  // lanes along the line: a warp stores contiguous outputs
    tl = uu / ng;
    ar = (uu % ng) * TOEP_RB;
  } else {       // lanes across lines: each of the RB stores is coalesced over the warp
    tl = uu % nl;
    ar = (uu / nl) * TOEP_RB;
  }
}

// acc[r] = Σ_j g[|a+r-j|] · Xs[j][tl]  for r < RB.
__device__ __forceinline__ void toep_dot4(const double* Ts, const double* Xs, int64_t n, int TL, int tl, int64_t a,
                                          double* acc) {
  const double* tp = Ts + 1 + (n - 1) + a;  // tp[r - j] = g[|a + r - j|]
  double w0 = tp[0], w1 = tp[1], w2 = tp[2], w3 = tp[3];
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
  const double* xs = Xs + tl;
  const int nn = static_cast<int>(n);
#pragma unroll 4
  for (int j = 0; j < nn; ++j) {
    const double x = xs[j * TL];
    c0 = fma(w0, x, c0);
    c1 = fma(w1, x, c1);
    c2 = fma(w2, x, c2);
    c3 = fma(w3, x, c3);
    w3 = w2;
    w2 = w1;
    w1 = w0;
    w0 = tp[-(j + 1)];
  }
  acc[0] = c0;
  acc[1] = c1;
  acc[2] = c2;
  acc[3] = c3;
}

// Shared-memory doubles a tile needs: Ts + Xs.
__host__ __device__ inline int64_t toep_smem_doubles(int64_t n, int64_t TL) { return toep_ts_doubles(n) + n * TL; }

}  // namespace gsgpc
