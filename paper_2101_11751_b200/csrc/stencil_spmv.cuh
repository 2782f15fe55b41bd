// stencil_spmv.cuh — one output of the half-stencil SpMV  (W^T W v)[a]
//   = A[0][a] v[a] + Σ_{s≥1} ( A[s][a] v[a + o_s] + A[s][a − o_s] v[a − o_s] )
// over the offset-major half stencil A[s][node] (reference: SufficientStats::apply_wtw,
// interp.cpp:224-241, on the CSR of the same matrix).  Shared by the public SpMV / graph
// CG (operators.cu) and the persistent EFCG kernel (efcg_persistent.cu) so both paths
// sum in the same order.
//
// Partners outside [0, m) hit exactly-zero stencil entries, so only the range mask is
// needed.  The loads of U = 8 offsets are issued before their FMAs: at one warp-wide 8-byte
// load per offset a thread needs many independent DRAM reads in flight to cover HBM
// latency (measured on B200: 75 → 50 µs per 173 MB stencil pass versus unroll 4).
#pragma once

#include "internal.cuh"

namespace gsgpc {

// OFF: functor s → o_s (a __constant__ table of the including translation unit).
//
// v is read with ld.global.ca (cached in L1): each element is read by the 2·S_min − 1
// neighbours around it, mostly by the same block.  This is also correct inside the
// persistent EFCG kernel, which rewrites v between grid barriers: grid.sync() invalidates
// L1 (CCTL.IVALL in the SASS).  Measured: config 3 SpMV phase 52 → 47.5 µs, config 5
// 102 → 91 µs, versus L2-only (ld.global.cg) loads.  The batched stencil loads are streaming
// (ld.global.cs, evict-first) — both the forward and the mirrored one: 47.6 → 44.8 µs
// (config 3), 90.5 → 86.2 µs (config 5); only one of the two streaming, or both
// ld.global.cg, measured no gain.
template <int SMIN, typename OFF, int U = 8>
__device__ __forceinline__ double stencil_row_dot(int m, const double* __restrict__ A, const double* __restrict__ v,
                                                  int a, OFF off) {
  auto ldv = [&](int i) -> double { return __ldca(v + i); };
  double acc0 = __ldg(A + a) * ldv(a), acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
  int s = 1;
  for (; s + U <= SMIN; s += U) {
    double af[U], ab[U], vf[U], vb[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int o = off(s + q);
      const int f = a + o, b = a - o;
      const bool okf = static_cast<unsigned>(f) < static_cast<unsigned>(m);
      const bool okb = static_cast<unsigned>(b) < static_cast<unsigned>(m);
      const double* As = A + static_cast<int64_t>(s + q) * m;
      af[q] = __ldcs(As + a);
      ab[q] = okb ? __ldcs(As + b) : 0.0;
      vf[q] = okf ? ldv(f) : 0.0;
      vb[q] = okb ? ldv(b) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < U; q += 2) {
      acc0 = fma(af[q], vf[q], acc0);
      acc1 = fma(ab[q], vb[q], acc1);
      acc2 = fma(af[q + 1], vf[q + 1], acc2);
      acc3 = fma(ab[q + 1], vb[q + 1], acc3);
    }
  }
  for (; s < SMIN; ++s) {
    const int o = off(s);
    const int f = a + o, b = a - o;
    const double* As = A + static_cast<int64_t>(s) * m;
    if (static_cast<unsigned>(f) < static_cast<unsigned>(m)) acc0 = fma(__ldg(As + a), ldv(f), acc0);
    if (static_cast<unsigned>(b) < static_cast<unsigned>(m)) acc1 = fma(__ldg(As + b), ldv(b), acc1);
  }
  return (acc0 + acc1) + (acc2 + acc3);
}

}  // namespace gsgpc
