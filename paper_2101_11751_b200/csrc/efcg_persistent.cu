// efcg_persistent.cu — the whole factorized_cg_grid_rhs loop (solvers.cpp:271-336) as ONE
// cooperative kernel: update → stencil SpMV + ρ → d Toeplitz mode products → fused
// epilogue + pap, separated by grid-wide barriers.  α, β, ρ, pap never leave the device;
// every block reduces the per-block partials itself in the same fixed order, so all blocks
// hold bit-identical scalars without an extra barrier.  Replaces the per-iteration chain of
// 2 + d kernel launches (launch gaps dominated the m ≈ 1e5 iteration).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "internal.cuh"
#include "precompute.cuh"
#include "stencil_spmv.cuh"
#include "toeplitz.cuh"

namespace cg = cooperative_groups;

namespace gsgpc {

constexpr int PCG_NT = 256;
#ifndef PCG_SPMV_U
#define PCG_SPMV_U 8  // offsets per load batch in the SpMV phase
#endif
#ifndef PCG_MINB
#define PCG_MINB 2  // resident blocks per SM (register cap 65536 / (256 · MINB))
#endif

struct PcgMode {
  int64_t n, inner, L;
  int TL, TA;
  int64_t tiles, chunks;
  const double* gen;
  int mm_stride, mm_cw, mm_ach;  // pcg_mode_mma: staged line stride, column tiles and row tiles per block task
  int mm_tz;                     // offset (doubles) of this mode's mirrored generator in shared memory
};

struct PcgArgs {
  int m;
  int d;
  const double* A;
  double *r, *u, *s, *z, *x, *t0, *t1;
  double *part_a, *part_b;
  double *trace, *alphas, *betas;
  CgState* st;
  PcgMode mode[3];
  int init;
  int plane;  // d = 3: modes 2 and 1 fused per x0-plane (pcg_plane_modes)
  int mma;    // Toeplitz modes on the FP64 tensor cores (pcg_mode_mma)
  int mm_xs;  // shared-memory offset (doubles) of the staged lines; the generators sit below it
  int mm_plane;              // d = 3: modes 2 and 1 fused per x0-plane on the tensor cores (pcg_plane_mma)
  int mp_parts, mp_ys;       // pcg_plane_mma: parts per plane, row stride of the mode-2 image
  unsigned long long* tbuf;  // optional phase trace: tbuf[iter * 8 + phase] = %globaltimer (ns)
  int off[kMaxSmin];         // flat stencil offsets o_s (per launch: no module-global table)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Sum of the per-block partials, identical in every block (fixed order, one warp).
__device__ __forceinline__ double grid_reduce(const double* part, int np, double* sh1) {
  if (threadIdx.x < 32) {
    double v = 0.0;
    for (int i = threadIdx.x; i < np; i += 32) v += __ldcg(part + i);
    v = warp_sum(v);
    if (threadIdx.x == 0) *sh1 = v;
  }
  __syncthreads();
  const double r = *sh1;
  __syncthreads();
  return r;
}

struct PcgOff {
  const int* o;  // → PcgArgs::off of the launch's __grid_constant__ parameter
  __device__ __forceinline__ int operator()(int s) const { return o[s]; }
};

template <int SMIN>
__device__ __forceinline__ double pcg_spmv_node(int m, const double* __restrict__ A, const double* __restrict__ v,
                                                int a, const int* off) {
  return stencil_row_dot<SMIN, PcgOff, PCG_SPMV_U>(m, A, v, a, PcgOff{off});
}

// One Toeplitz mode product (grid-stride over line tiles × output chunks).  EPI: fused
// v̂ = (K û) + σ² r̂, ŝ = û + β ŝ, z̄ = v̂ + β z̄ and the ŝ·z̄ partial.
template <bool EPI>
__device__ __forceinline__ void pcg_mode(const PcgMode& c, const double* X, double* Y, double* smem,
                                         const PcgArgs& a, double beta, double s2, double& dot) {
  const int64_t n = c.n;
  double* Ts = smem;
  double* Xs = smem + toep_ts_doubles(n);
  const int64_t nwork = c.tiles * c.chunks;
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int64_t tile = w % c.tiles, chunk = w / c.tiles;
    const int64_t l0 = tile * c.TL;
    const int nl = static_cast<int>(imin64(c.TL, c.L - l0));
    const int64_t a0 = chunk * c.TA;
    const int na = static_cast<int>(imin64(c.TA, n - a0));
    __syncthreads();
    toep_load_tile(X, c.gen, n, c.inner, c.TL, l0, nl, Ts, Xs, PCG_NT);
    __syncthreads();
    const int ngroups = nl * ((na + TOEP_RB - 1) / TOEP_RB);
    for (int uu = threadIdx.x; uu < ngroups; uu += PCG_NT) {
      int tl, ar;
      toep_group(uu, nl, na, c.inner == 1, tl, ar);
      const int64_t l = l0 + tl, o = l / c.inner, i = l % c.inner;
      // epilogue operands issued before the dot so their latency hides under it
      double er[TOEP_RB], eu[TOEP_RB], es[TOEP_RB], ez[TOEP_RB];
      if (EPI) {
#pragma unroll
        for (int r = 0; r < TOEP_RB; ++r) {
          const bool ok = ar + r < na;
          const int64_t g = (o * n + a0 + ar + r) * c.inner + i;
          er[r] = ok ? __ldcg(a.r + g) : 0.0;
          eu[r] = ok ? __ldcg(a.u + g) : 0.0;
          es[r] = ok ? __ldcg(a.s + g) : 0.0;
          ez[r] = ok ? __ldcg(a.z + g) : 0.0;
        }
      }
      double acc[TOEP_RB];
      toep_dot4(Ts, Xs, n, c.TL, tl, a0 + ar, acc);
#pragma unroll
      for (int r = 0; r < TOEP_RB; ++r) {
        if (ar + r >= na) break;
        const int64_t g = (o * n + a0 + ar + r) * c.inner + i;
        if (!EPI) {
          Y[g] = acc[r];
        } else {
          const double v = acc[r] + s2 * er[r];
          const double sn = eu[r] + beta * es[r];
          const double zn = v + beta * ez[r];
          a.s[g] = sn;
          a.z[g] = zn;
          dot = fma(sn, zn, dot);
        }
      }
    }
  }
}

// One Toeplitz mode on the FP64 tensor cores (mma.sync.m8n8k4.f64).  A block task = 8·CW
// lines × ACH row tiles: the block stages the lines in shared memory with all its threads
// (many loads in flight), then each warp item (8 lines × 8 outputs) accumulates
// D[a][line] = Σ_j T[a − j] · X(line, j) over j in k-steps of 4 — A = an 8 × 4 tile of the
// Toeplitz matrix from the mirrored generator Tz, B = 4 positions × 8 staged lines — in two
// independent accumulator chains (even / odd k-steps).  The CUDA-core tile kernel ran one
// 4-output dot of length n per thread on ~L·n/1024 blocks (config 2's 256-node modes: 72 busy
// blocks, ~12–17 µs per mode).
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__host__ __device__ inline int64_t mm_gen_doubles(int64_t n) { return 2 * n + 12; }
// staged line stride ≡ 4 (mod 16) doubles: the B-fragment loads (8 lines × 4 positions) hit
// every bank pair twice — 2 wavefronts per 32 doubles
__host__ __device__ inline int64_t mm_stride(int64_t n) {
  const int64_t n4 = (n + 3) & ~int64_t{3};
  return n4 + ((4 - n4 % 16) + 16) % 16;
}

template <bool EPI>
__device__ __forceinline__ void pcg_mode_mma(const PcgMode& c, const double* X, double* Y, double* smem,
                                             const PcgArgs& a, double beta, double s2, double& dot) {
  const int n = static_cast<int>(c.n);
  const int64_t inner = c.inner, L = c.L;
  const int stride = c.mm_stride, CW = c.mm_cw, ACH = c.mm_ach;
  const double* Tz = smem + c.mm_tz;  // written once at kernel start (pcg_mma_gens)
  double* Xs = smem + a.mm_xs;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, r8 = lane >> 2, kq = lane & 3;
  const int nat = (n + 7) >> 3, nk = (n + 3) >> 2, n4 = 4 * nk;
  const int TLN = 8 * CW;
  const int64_t nlb = (L + TLN - 1) / TLN;
  const int nac = (nat + ACH - 1) / ACH;
  const int64_t ntask = nlb * nac;
  for (int64_t task = blockIdx.x; task < ntask; task += gridDim.x) {
    const int64_t lb = task / nac;
    const int ac = static_cast<int>(task - lb * nac);
    const int64_t l0 = lb * TLN;
    const int nl = static_cast<int>(imin64(TLN, L - l0));
    __syncthreads();  // previous task's Xs consumed
    // stage lines [l0, l0 + nl) × positions [0, n4) (zeros past n and past the last line)
    const int cnt = TLN * n4;
    for (int q0 = threadIdx.x; q0 < cnt; q0 += 8 * PCG_NT) {
      double t[8];
      int dst[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int q = q0 + u * PCG_NT;
        int ln, j;
        if (inner == 1) {  // lines contiguous: positions fastest
          ln = q / n4;
          j = q - ln * n4;
        } else {           // positions strided by inner: lines fastest (coalesced)
          j = q / TLN;
          ln = q - j * TLN;
        }
        dst[u] = q < cnt ? ln * stride + j : -1;
        const int64_t l = l0 + ln;
        const bool ok = q < cnt && ln < nl && j < n;
        const int64_t lo = l / inner, li = l - lo * inner;
        t[u] = ok ? __ldcg(X + (lo * n + j) * inner + li) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (dst[u] >= 0) Xs[dst[u]] = t[u];
    }
    __syncthreads();
    const int at0 = ac * ACH;
    const int na = min(ACH, nat - at0);
    for (int it = warp; it < CW * na; it += PCG_NT / 32) {
      const int cw = it % CW, at = at0 + it / CW;
      const double* xs = Xs + (cw * 8 + r8) * stride + kq;
      const double* tz = Tz + (n + 3) + at * 8 + r8 - kq;
      const int aa = at * 8 + r8;
      // epilogue operands issued before the k-loop (their latency hides under the MMAs)
      int64_t gi[2] = {-1, -1};
      double er[2] = {0.0, 0.0}, eu[2] = {0.0, 0.0}, es[2] = {0.0, 0.0}, ez[2] = {0.0, 0.0};
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int lc = cw * 8 + 2 * kq + e;
        if (aa < n && lc < nl) {
          const int64_t ll = l0 + lc;
          const int64_t oo = ll / inner, ii = ll - oo * inner;
          gi[e] = (oo * n + aa) * inner + ii;
          if (EPI) {
            er[e] = __ldcg(a.r + gi[e]);
            eu[e] = __ldcg(a.u + gi[e]);
            es[e] = __ldcg(a.s + gi[e]);
            ez[e] = __ldcg(a.z + gi[e]);
          }
        }
      }
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
      int s = 0;
      for (; s + 1 < nk; s += 2) {
        dmma(d0, d1, tz[-4 * s], xs[4 * s]);
        dmma(e0, e1, tz[-4 * (s + 1)], xs[4 * (s + 1)]);
      }
      if (s < nk) dmma(d0, d1, tz[-4 * s], xs[4 * s]);
      const double acc[2] = {d0 + e0, d1 + e1};
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t g = gi[e];
        if (g < 0) continue;
        if (!EPI) {
          Y[g] = acc[e];
        } else {
          const double v = acc[e] + s2 * er[e];
          const double sn = eu[e] + beta * es[e];
          const double zn = v + beta * ez[e];
          a.s[g] = sn;
          a.z[g] = zn;
          dot = fma(sn, zn, dot);
        }
      }
    }
  }
}

// One warp item of a tensor-core mode product from shared memory: D[a][col] for the 8 rows
// a = at·8 + r8 and the 8 columns of the tile, D = Σ_j T[a − j] · B(j, col), with
// B(j, col) = xs[j · js + col · cs] (j = 4 s + kq, col = r8 for the fragment load).
__device__ __forceinline__ void mm_item(const double* Tz, int n, int at, const double* xs, int js, int cs, int r8,
                                        int kq, double* acc) {
  const double* tz = Tz + (n + 3) + at * 8 + r8 - kq;
  const double* xb = xs + kq * js + r8 * cs;
  const int nk = (n + 3) >> 2;
  double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
  int s = 0;
  for (; s + 1 < nk; s += 2) {
    dmma(d0, d1, tz[-4 * s], xb[4 * s * js]);
    dmma(e0, e1, tz[-4 * (s + 1)], xb[4 * (s + 1) * js]);
  }
  if (s < nk) dmma(d0, d1, tz[-4 * s], xb[4 * s * js]);
  acc[0] = d0 + e0;
  acc[1] = d1 + e1;
}

// d = 3, tensor cores: modes 2 and 1 of K_G û in ONE grid phase.  Task = (x0-plane p, part):
// stage the plane X[i1][i2] (row stride mm_stride(n2), zero-padded), mode 2 over all of it
// into Y[i1][a2] (row stride mp_ys ≡ 8 mod 16 so the mode-1 fragment loads are
// conflict-free), then mode 1 for the part's a1 row tiles → t0.  Each part redoes the
// plane's mode 2 (n1·n2² MACs, a few hundred MMAs) instead of paying a grid barrier and a
// second phase.
__device__ __forceinline__ void pcg_plane_mma(const PcgArgs& a, double* smem) {
  const PcgMode &c1 = a.mode[1], &c2 = a.mode[2];
  const int n0 = static_cast<int>(a.mode[0].n), n1 = static_cast<int>(c1.n), n2 = static_cast<int>(c2.n);
  const int xs_st = c2.mm_stride, ys_st = a.mp_ys, P = a.mp_parts;
  const int n1p = (n1 + 7) & ~7, n2p4 = (n2 + 3) & ~3, n1p4 = (n1 + 3) & ~3;
  const double* T2 = smem + c2.mm_tz;
  const double* T1 = smem + c1.mm_tz;
  double* X = smem + a.mm_xs;
  double* Y = X + static_cast<int64_t>(n1p) * xs_st;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, r8 = lane >> 2, kq = lane & 3;
  const int nat1 = (n1 + 7) >> 3, nat2 = (n2 + 7) >> 3, nlt2 = n1p >> 3, nlt1 = (n2 + 7) >> 3;
  for (int task = blockIdx.x; task < n0 * P; task += gridDim.x) {
    const int p = task / P, part = task - p * P;
    const double* src = a.u + static_cast<int64_t>(p) * n1 * n2;
    __syncthreads();
    // stage rows i1 < n1p, positions < n2p4 (zeros outside the plane)
    const int cnt = n1p * n2p4;
    for (int q0 = threadIdx.x; q0 < cnt; q0 += 8 * PCG_NT) {
      double t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int q = q0 + u * PCG_NT;
        const int i1 = q / n2p4, i2 = q - i1 * n2p4;
        t[u] = (q < cnt && i1 < n1 && i2 < n2) ? __ldcg(src + i1 * n2 + i2) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int q = q0 + u * PCG_NT;
        const int i1 = q / n2p4, i2 = q - i1 * n2p4;
        if (q < cnt) X[i1 * xs_st + i2] = t[u];
      }
    }
    // Y rows past n1 (read as zero positions by mode 1)
    for (int q = threadIdx.x; q < (n1p4 - n1) * ys_st; q += PCG_NT) Y[n1 * ys_st + q] = 0.0;
    __syncthreads();
    // mode 2: lines i1 (columns), positions i2 → Y[i1][a2]
    for (int it = warp; it < nlt2 * nat2; it += PCG_NT / 32) {
      const int lt = it / nat2, at = it - lt * nat2;
      double acc[2];
      mm_item(T2, n2, at, X + lt * 8 * xs_st, 1, xs_st, r8, kq, acc);
      const int a2 = at * 8 + r8;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i1 = lt * 8 + 2 * kq + e;
        if (a2 < n2) Y[i1 * ys_st + a2] = acc[e];  // rows ≥ n1 hold zeros' images (0)
      }
    }
    __syncthreads();
    // mode 1 for this part's a1 row tiles: lines i2 (columns), positions i1 → t0[p][a1][i2]
    const int q_lo = part * nat1 / P, q_hi = (part + 1) * nat1 / P;
    double* dst = a.t0 + static_cast<int64_t>(p) * n1 * n2;
    for (int it = warp; it < nlt1 * (q_hi - q_lo); it += PCG_NT / 32) {
      const int lt = it % nlt1, at = q_lo + it / nlt1;
      double acc[2];
      mm_item(T1, n1, at, Y + lt * 8, ys_st, 1, r8, kq, acc);
      const int a1 = at * 8 + r8;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i2 = lt * 8 + 2 * kq + e;
        if (a1 < n1 && i2 < n2) dst[a1 * n2 + i2] = acc[e];
      }
    }
  }
}

// d = 3: the last two Toeplitz modes of K_G û in ONE grid phase.  Work item = (x0-plane p,
// part q of the plane's x1 outputs): the block stages the plane (n1 × n2) in shared memory,
// applies mode 2 to all of it, then mode 1 for its x1 outputs only — the plane's mode 2 is
// recomputed by each of its parts, which is cheaper than a grid barrier and a second
// phase (each part has ~n1·n2·n2 + n1·n2·n1/P FMAs).  Sums run in the order of toep_dot4
// (j ascending), so results equal the two-phase path bit for bit.
// Σ_j T[a + r − j] · x(j), r < 4, over j = 0..n−1 in order (toep_dot4's sliding window);
// T = Ts + 1 + (n − 1) of a zero-padded mirrored generator (toep_ts_doubles(n) doubles).
template <typename X>
__device__ __forceinline__ void plane_dot4(const double* Ts, int n, int a, X x, double* acc) {
  const double* tp = Ts + 1 + (n - 1) + a;
  double w0 = tp[0], w1 = tp[1], w2 = tp[2], w3 = tp[3];
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
#pragma unroll 4
  for (int j = 0; j < n; ++j) {
    const double v = x(j);
    c0 = fma(w0, v, c0);
    c1 = fma(w1, v, c1);
    c2 = fma(w2, v, c2);
    c3 = fma(w3, v, c3);
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

__device__ __forceinline__ void plane_gen(double* Ts, const double* g, int n) {
  if (threadIdx.x < 5) Ts[threadIdx.x == 0 ? 0 : 2 * n - 1 + threadIdx.x] = 0.0;
  for (int q = threadIdx.x; q < 2 * n - 1; q += PCG_NT) Ts[1 + q] = g[abs(q - (n - 1))];
}

__device__ __forceinline__ void pcg_plane_modes(const PcgArgs& a, double* smem) {
  const int n0 = static_cast<int>(a.mode[0].n), n1 = static_cast<int>(a.mode[1].n), n2 = static_cast<int>(a.mode[2].n);
  const int pl = n1 * n2;
  const int g2 = (n2 + 3) >> 2, g1 = (n1 + 3) >> 2;  // 4-output groups per line
  const int P = max(1, min(g1, static_cast<int>(gridDim.x) / n0));  // parts per plane
  double* T2 = smem;
  double* T1 = T2 + toep_ts_doubles(n2);
  double* X = T1 + toep_ts_doubles(n1);
  double* Y = X + pl;
  __syncthreads();
  plane_gen(T2, a.mode[2].gen, n2);
  plane_gen(T1, a.mode[1].gen, n1);
  for (int w = blockIdx.x; w < n0 * P; w += gridDim.x) {
    const int p = w / P, part = w - p * P;
    const double* src = a.u + static_cast<int64_t>(p) * pl;
    __syncthreads();
    for (int i0 = threadIdx.x; i0 < pl; i0 += 8 * PCG_NT) {  // 8 loads in flight per thread
      double t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) t[u] = i0 + u * PCG_NT < pl ? __ldcg(src + i0 + u * PCG_NT) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i0 + u * PCG_NT < pl) X[i0 + u * PCG_NT] = t[u];
    }
    __syncthreads();
    // mode 2 over the whole plane: Y[i1][a2]
    for (int o = threadIdx.x; o < n1 * g2; o += PCG_NT) {
      const int i1 = o / g2, ar = (o - i1 * g2) * 4;
      const double* xr = X + i1 * n2;
      double acc[4];
      plane_dot4(T2, n2, ar, [&](int j) { return xr[j]; }, acc);
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (ar + r < n2) Y[i1 * n2 + ar + r] = acc[r];
    }
    __syncthreads();
    // mode 1 for this part's x1 outputs (groups of 4 consecutive a1 per column i2)
    const int q_lo = part * g1 / P, q_hi = (part + 1) * g1 / P;
    double* dst = a.t0 + static_cast<int64_t>(p) * pl;
    for (int o = threadIdx.x; o < (q_hi - q_lo) * n2; o += PCG_NT) {
      const int gq = q_lo + o / n2, i2 = o - (o / n2) * n2;
      const int ar = gq * 4;
      double acc[4];
      plane_dot4(T1, n1, ar, [&](int j) { return Y[j * n2 + i2]; }, acc);
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (ar + r < n1) dst[(ar + r) * n2 + i2] = acc[r];
    }
  }
}

template <int SMIN>
__global__ void __launch_bounds__(PCG_NT, PCG_MINB) k_efcg_persistent(const __grid_constant__ PcgArgs a) {
  extern __shared__ double smem[];
  __shared__ double sh[8];
  __shared__ double sh1;
  cg::grid_group grid = cg::this_grid();
  CgState* st = a.st;
  const double s2 = st->sigma_sq;
  const int maxiter = st->maxiter;
  double rho = st->rho, pap = st->pap, eps = st->eps;
  int iter = st->iter;
  int converged = 0, breakdown = 0;
  const int m = a.m;
  const int tid = blockIdx.x * PCG_NT + threadIdx.x;
  const int nthr = gridDim.x * PCG_NT;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  if (a.mma) {  // mirrored generators of every mode, resident for the whole solve
    for (int k = 0; k < a.d; ++k) {
      const int n = static_cast<int>(a.mode[k].n);
      double* Tz = smem + a.mode[k].mm_tz;  // Tz[(n + 3) + q] = g[|q|] for |q| < n, else 0
      for (int q = threadIdx.x; q < mm_gen_doubles(n); q += PCG_NT) {
        const int dq = q - (n + 3);
        const int ad = dq < 0 ? -dq : dq;
        Tz[q] = ad < n ? a.mode[k].gen[ad] : 0.0;
      }
    }
    __syncthreads();
  }

  auto spmv_phase = [&]() {
    double dot = 0.0;
    for (int node = tid; node < m; node += nthr) {
      const double u = pcg_spmv_node<SMIN>(m, a.A, a.r, node, a.off);
      a.u[node] = u;
      dot = fma(u, __ldcg(a.r + node), dot);
    }
    const double bs = block_sum<PCG_NT>(dot, sh);
    if (threadIdx.x == 0) a.part_a[blockIdx.x] = bs;
  };
  auto stamp = [&](int phase) {
    if (a.tbuf && leader && iter < 64) a.tbuf[iter * 8 + phase] = gtimer();
  };
  auto kg_phase = [&](double beta) {
    double dot = 0.0;
    const double* src = a.u;
    int k_top = a.d - 1;
    if (a.mma) {
      if (a.mm_plane) {
        pcg_plane_mma(a, smem);
        grid.sync();
        stamp(3);
        src = a.t0;
        k_top = 0;
      }
      for (int k = k_top; k >= 1; --k) {
        double* dst = (src == a.t0) ? a.t1 : a.t0;
        pcg_mode_mma<false>(a.mode[k], src, dst, smem, a, beta, s2, dot);
        grid.sync();
        stamp(5 - k);
        src = dst;
      }
      pcg_mode_mma<true>(a.mode[0], src, nullptr, smem, a, beta, s2, dot);
      const double bs = block_sum<PCG_NT>(dot, sh);
      if (threadIdx.x == 0) a.part_b[blockIdx.x] = bs;
      return;
    }
    if (a.plane) {
      pcg_plane_modes(a, smem);
      grid.sync();
      stamp(3);
      src = a.t0;
      k_top = 0;
    }
    for (int k = k_top; k >= 1; --k) {
      double* dst = (src == a.t0) ? a.t1 : a.t0;
      pcg_mode<false>(a.mode[k], src, dst, smem, a, beta, s2, dot);
      grid.sync();
      stamp(5 - k);
      src = dst;
    }
    pcg_mode<true>(a.mode[0], src, nullptr, smem, a, beta, s2, dot);
    const double bs = block_sum<PCG_NT>(dot, sh);
    if (threadIdx.x == 0) a.part_b[blockIdx.x] = bs;
  };

  if (a.init) {
    spmv_phase();
    grid.sync();
    rho = grid_reduce(a.part_a, gridDim.x, &sh1);
    eps = st->eps_abs >= 0.0 ? st->eps_abs : st->rel_tol * st->rel_tol * rho;
    if (leader) a.trace[0] = rho;
    if (rho <= eps) {
      converged = 1;
    } else {
      kg_phase(0.0);
      grid.sync();
      pap = grid_reduce(a.part_b, gridDim.x, &sh1);
    }
  }
  while (!converged) {
    if (iter >= maxiter) break;
    if (pap <= 0.0) {
      breakdown = 1;
      break;
    }
    const double alpha = rho / pap;
    stamp(0);
    // ŝ, z̄ were written by other blocks (L2 loads); 4 elements per thread in flight
    for (int i0 = tid; i0 < m; i0 += 4 * nthr) {
      double sv[4], zv[4], xv[4], rv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * nthr;
        const bool in = i < m;
        sv[u] = in ? __ldcg(a.s + i) : 0.0;
        zv[u] = in ? __ldcg(a.z + i) : 0.0;
        xv[u] = in ? a.x[i] : 0.0;
        rv[u] = in ? a.r[i] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * nthr;
        if (i < m) {
          a.x[i] = xv[u] + alpha * sv[u];
          a.r[i] = rv[u] - alpha * zv[u];
        }
      }
    }
    if (leader) a.alphas[iter] = alpha;
    grid.sync();
    stamp(1);
    spmv_phase();
    grid.sync();
    stamp(2);
    const double rho_new = grid_reduce(a.part_a, gridDim.x, &sh1);
    ++iter;
    if (leader) a.trace[iter] = rho_new;
    if (rho_new <= eps) {
      converged = 1;
      rho = rho_new;
      break;
    }
    const double beta = rho_new / rho;
    if (leader) a.betas[iter - 1] = beta;
    rho = rho_new;
    --iter;
    kg_phase(beta);
    grid.sync();
    stamp(6);
    ++iter;
    pap = grid_reduce(a.part_b, gridDim.x, &sh1);
  }
  if (leader) {
    st->rho = rho;
    st->pap = pap;
    st->eps = eps;
    st->iter = iter;
    st->converged = converged;
    st->breakdown = breakdown;
    st->done = 1;
  }
}

static PcgMode mode_cfg(const KgDev& kg, int k) {
  PcgMode c{};
  int64_t inner = 1, outer = 1;
  for (int j = k + 1; j < kg.d; ++j) inner *= kg.sz[j];
  for (int j = 0; j < k; ++j) outer *= kg.sz[j];
  const int64_t n = kg.sz[k];
  c.n = n;
  c.inner = inner;
  c.L = inner * outer;
  const int64_t cap = 6144;  // doubles of dynamic smem per block (48 KB)
  if (toep_smem_doubles(n, 1) > cap) {
    throw Error(GSGPC_UNSUPPORTED, "K_G: grid dimension larger than 2040 nodes is not supported");
  }
  int64_t TL = std::min<int64_t>(32, (cap - toep_ts_doubles(n)) / n);
  TL = std::max<int64_t>(1, std::min<int64_t>(TL, c.L));
  c.TL = static_cast<int>(TL);
  c.tiles = ceil_div(c.L, TL);
  int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(1184, c.tiles), ceil_div(n, 32)));
  c.TA = static_cast<int>(ceil_div(n, chunks));
  c.chunks = ceil_div(n, c.TA);
  c.gen = kg.gen[k];
  return c;
}

// Launch of the persistent kernel.  The function attributes (dynamic shared-memory limit and
// the shared-memory carveout) belong to the kernel, not to a launch, so they are set before
// EVERY launch — a solve with another shared-memory size in between (another grid, another
// context on the device) would otherwise leave a carveout under which the cached grid no longer
// fits ("too many blocks in cooperative launch") — and attribute setting + launch run under one
// lock per kernel instantiation.  The grid size per (device, dynamic smem) is cached.
template <int SMIN>
static void launch_pcg(const Launch& L, const PcgArgs& a, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, size_t>, int> cache;
  int dev = 0;
  GSGPC_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  GSGPC_CUDA(cudaFuncSetAttribute(k_efcg_persistent<SMIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(std::max<size_t>(smem, 48 * 1024))));
  // smallest shared-memory carveout that holds the resident blocks: the rest is L1
  const int pct =
      static_cast<int>(std::min<size_t>(100, (PCG_MINB * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024)));
  GSGPC_CUDA(cudaFuncSetAttribute(k_efcg_persistent<SMIN>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
  int grid = 0;
  auto it = cache.find({dev, smem});
  if (it != cache.end()) {
    grid = it->second;
  } else {
    int sms = 0, per_sm = 0;
    GSGPC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    GSGPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_efcg_persistent<SMIN>, PCG_NT, smem));
    if (per_sm < 1) throw Error(GSGPC_CUDA_ERROR, "persistent EFCG kernel cannot be resident");
    grid = sms * std::min(per_sm, 4);
    cache[{dev, smem}] = grid;
  }
  // small grids: about one node per thread, at least 32 blocks — every grid barrier costs
  // more with more blocks (config 1, m = 1000: 296 blocks 0.064, 32 blocks 0.032 ms/iteration;
  // 16 blocks 0.048)
  int nblk = std::min<int>(grid, std::max<int>(32, static_cast<int>(ceil_div(a.m, PCG_NT))));
  static const int force = [] {  // diagnostics: GSGPC_CG_BLOCKS = persistent grid size
    const char* e = getenv("GSGPC_CG_BLOCKS");
    return e ? atoi(e) : 0;
  }();
  if (force > 0) nblk = std::min(grid, force);
  PcgArgs aa = a;
  void* params[] = {&aa};
  GSGPC_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_efcg_persistent<SMIN>), dim3(nblk), dim3(PCG_NT),
                                         params, smem, L.s));
  L.count();
}

void run_efcg_persistent(const Launch& L, const StencilDesc& sd, const double* A, const KgDev& kg, const CgBufs& b,
                         int init, unsigned long long* tbuf) {
  PcgArgs a{};
  {
    const StencilOffsets off = make_stencil_offsets(sd);
    for (int s2 = 0; s2 < sd.S_min; ++s2) a.off[s2] = off.o32[s2];
  }
  a.m = static_cast<int>(sd.m);
  a.d = sd.d;
  a.A = A;
  a.r = b.r;
  a.u = b.u;
  a.s = b.s;
  a.z = b.z;
  a.x = b.x;
  a.t0 = b.kt0;
  a.t1 = b.kt1;
  a.part_a = b.part_a;
  a.part_b = b.part_b;
  a.trace = b.trace;
  a.alphas = b.alphas;
  a.betas = b.betas;
  a.st = b.st;
  a.init = init;
  a.tbuf = tbuf;
  size_t smem = 0;
  for (int k = 0; k < kg.d; ++k) {
    a.mode[k] = mode_cfg(kg, k);
    smem = std::max(smem, sizeof(double) * static_cast<size_t>(toep_smem_doubles(a.mode[k].n, a.mode[k].TL)));
  }
  // FP64 tensor-core modes whenever every mode has enough lines to fill the grid (d ≥ 2 at
  // the BASELINE sizes; d = 1 has a single line).  GSGPC_CG_TOEP_SIMT=1: the CUDA-core tiles.
  static const bool simt = [] {
    const char* e = getenv("GSGPC_CG_TOEP_SIMT");
    return e && e[0] == '1';
  }();
  bool mma = !simt && kg.d >= 2;
  int64_t gens = 0;
  for (int k = 0; k < kg.d; ++k) gens += mm_gen_doubles(a.mode[k].n);
  size_t mm_smem = 0;
  for (int k = 0, tz = 0; k < kg.d && mma; ++k) {
    PcgMode& c = a.mode[k];
    const int64_t st = mm_stride(c.n);
    const int64_t cwmax = std::min<int64_t>(8, (6144 - gens) / (8 * st));
    if (c.L < 64 || cwmax < 1) {
      mma = false;
      break;
    }
    const int64_t target = PCG_MINB * sm_count();  // one block task per resident block, one wave
    const int64_t nlt = ceil_div(c.L, 8);
    const int64_t cw = std::max<int64_t>(1, std::min<int64_t>(cwmax, ceil_div(nlt, target)));
    const int64_t nlb = ceil_div(nlt, cw);
    const int64_t nat = ceil_div(c.n, 8);
    const int64_t nac = std::max<int64_t>(1, std::min<int64_t>(nat, target / nlb));
    c.mm_stride = static_cast<int>(st);
    c.mm_cw = static_cast<int>(cw);
    c.mm_ach = static_cast<int>(ceil_div(nat, nac));
    c.mm_tz = tz;
    tz += static_cast<int>(mm_gen_doubles(c.n));
    mm_smem = std::max(mm_smem, sizeof(double) * static_cast<size_t>(gens + 8 * cw * st));
  }
  a.mm_xs = static_cast<int>(gens);
  size_t mp_smem = 0;
  if (mma && kg.d == 3 && !getenv("GSGPC_CG_NOPLANE")) {
    // plane fusion of modes 2 and 1 when the staged plane and its mode-2 image fit in 48 KB
    // per block.  Measured (B200, per iteration): config 3 (80·20-node planes) modes
    // 23.6 → 18.9 µs; config 5 (64·64-node planes, 75 KB) 25.3 → 26.2 µs — there every part
    // re-stages and re-transforms a 4096-node plane, more than the saved barrier.
    const int64_t n0 = a.mode[0].n, n1 = a.mode[1].n, n2 = a.mode[2].n;
    const int64_t n1p = (n1 + 7) & ~int64_t{7}, n1p4 = (n1 + 3) & ~int64_t{3};
    const int64_t ys = ((n2 + 7) & ~int64_t{7}) + ((((n2 + 7) & ~int64_t{7}) % 16) == 0 ? 8 : 0);
    const int64_t need = gens + n1p * mm_stride(n2) + std::max(n1p, n1p4) * ys;
    static const int64_t plane_kb = [] {  // diagnostics: shared-memory budget of the plane phase
      const char* e = getenv("GSGPC_CG_PLANE_KB");
      return e ? static_cast<int64_t>(atoi(e)) : int64_t{48};
    }();
    if (need * 8 <= plane_kb * 1024) {
      a.mm_plane = 1;
      a.mp_ys = static_cast<int>(ys);
      a.mp_parts = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n1, 8), PCG_MINB * sm_count() / n0)));
      if (const char* e = getenv("GSGPC_CG_PLANE_PARTS")) a.mp_parts = std::max(1, atoi(e));  // diagnostics
      mp_smem = static_cast<size_t>(need * 8);
    }
  }
  // the tensor-core path needs only its own shared memory (generators + staged lines /
  // plane): the rest of the SM's 256 KB stays L1, which serves the SpMV's vector and
  // mirrored-stencil reads
  if (mma) smem = std::max(mm_smem, a.mm_plane ? mp_smem : size_t{0});
  if (mma) {
    a.mma = 1;
  } else if (kg.d == 3 && !getenv("GSGPC_CG_NOPLANE")) {  // GSGPC_CG_NOPLANE=1: three mode phases (diagnostics)
    const int64_t n1 = a.mode[1].n, n2 = a.mode[2].n;
    const int64_t need = toep_ts_doubles(n1) + toep_ts_doubles(n2) + 2 * n1 * n2;
    if (need <= 6144) {
      a.plane = 1;
      smem = std::max(smem, sizeof(double) * static_cast<size_t>(need));
    }
  }
  switch (sd.S_min) {
    case 172: launch_pcg<172>(L, a, smem); break;
    case 25: launch_pcg<25>(L, a, smem); break;
    case 4: launch_pcg<4>(L, a, smem); break;
    case 14: launch_pcg<14>(L, a, smem); break;
    case 5: launch_pcg<5>(L, a, smem); break;
    default: launch_pcg<2>(L, a, smem); break;
  }
  GSGPC_CUDA(cudaGetLastError());
}

}  // namespace gsgpc
