// operators.cu — per-iteration operators of the factorized solvers.
//
//   K3  k_spmv / k_cg_spmv : W^T W as a symmetric 7^d (3^d linear) stencil SpMV over the
//                            regular grid (replaces SufficientStats::apply_wtw's CSR SpMV,
//                            interp.cpp:227-233).  Only the lexicographically non-negative
//                            half of the offsets is stored; the mirrored half is read at the
//                            shifted node (A[s][a-δ] x[a-δ]).
//   K4  k_toep             : K_G v as d Toeplitz mode products (K_G = ⊗_k T_k for the
//                            SE-ARD kernel, kernels.cpp:43-55), replacing the circulant-
//                            embedding FFT of ToeplitzOperator::apply (grid.cpp:193-235).
//   K5  k_cg_*             : fused EFCG vector updates with device-resident α, β, ρ, pap
//                            (factorized_cg_grid_rhs, solvers.cpp:271-336); dots use
//                            per-block partials + a last-block reduction (deterministic).
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "internal.cuh"
#include "precompute.cuh"
#include "stencil_spmv.cuh"
#include "toeplitz.cuh"

namespace gsgpc {

StencilOffsets make_stencil_offsets(const StencilDesc& sd) {
  StencilOffsets t{};
  const int E = 2 * sd.W - 1;
  int S = 1;
  for (int k = 0; k < sd.d; ++k) S *= E;
  const int c0 = (S - 1) / 2;
  for (int s2 = 0; s2 < sd.S_min; ++s2) {
    int q = c0 + s2;
    long long f = 0;
    int dig[3] = {0, 0, 0};
    for (int k = sd.d - 1; k >= 0; --k) {
      dig[k] = q % E - (sd.W - 1);
      q /= E;
    }
    for (int k = 0; k < sd.d; ++k) {
      f = f * sd.sz[k] + dig[k];
      t.d[s2][k] = static_cast<signed char>(dig[k]);
    }
    t.flat[s2] = f;
    t.o32[s2] = static_cast<int>(f);
  }
  return t;
}

PencilTables make_pencil_tables(const StencilDesc& sd) {
  PencilTables t{};
  const int E = 2 * sd.W - 1;
  int S = 1;
  for (int k = 0; k < sd.d; ++k) S *= E;
  const int c0 = (S - 1) / 2;
  int npen = 1;
  for (int k = 0; k + 1 < sd.d; ++k) npen *= E;
  for (int q = 0; q < npen; ++q) {
    int dig[3] = {0, 0, 0};
    int r = q;
    for (int k = sd.d - 2; k >= 0; --k) {
      dig[k] = r % E - (sd.W - 1);
      r /= E;
    }
    long long f = 0;
    for (int k = 0; k < sd.d; ++k) f = f * sd.sz[k] + (k + 1 < sd.d ? dig[k] : 0);
    t.ob[q] = static_cast<int>(f);
    for (int tt = 0; tt < E; ++tt) {
      int full = 0;
      for (int k = 0; k < sd.d; ++k) full = full * E + (k + 1 < sd.d ? dig[k] : tt - (sd.W - 1)) + (sd.W - 1);
      t.s[q][tt] = full >= c0 ? full - c0 : -((S - 1 - full) - c0) - 1;
    }
  }
  return t;
}

// ------------------------------------------------------------------ K3 stencil SpMV
// Check-free variant for the solvers' internal (finite) vectors.  With row-major
// flattening, a partner node outside the grid maps either outside [0, m) (masked) or to a
// stored entry that is exactly zero: the pair (a, a+δ) with a+δ off-grid is never touched
// by any point, and the mirrored read A[s][flat(a-δ)] with a-δ off-grid lands on a node b'
// whose own partner b'+δ is off-grid (else b' = a-δ would be on-grid).  So every thread runs
// the same unrolled loop (no divergence) and the blocks stay in step, which keeps the
// mirrored-half reads in L2.
struct OpOff {
  const int* o;  // → the launch's __grid_constant__ StencilOffsets::o32
  __device__ __forceinline__ int operator()(int s) const { return o[s]; }
};

template <int SMIN>
__device__ __forceinline__ double spmv_node_fast(int64_t m64, const double* __restrict__ A,
                                                 const double* __restrict__ v, int64_t a64, const int* o32) {
  // 32-bit indexing: S_min·m < 2^31 is checked on the host
  return stencil_row_dot<SMIN>(static_cast<int>(m64), A, v, static_cast<int>(a64), OpOff{o32});
}

__device__ __forceinline__ double spmv_node_any(const StencilDesc& sd, const double* __restrict__ A,
                                                const double* __restrict__ v, int64_t a, const int* o32) {
  switch (sd.S_min) {
    case 172: return spmv_node_fast<172>(sd.m, A, v, a, o32);
    case 25: return spmv_node_fast<25>(sd.m, A, v, a, o32);
    case 4: return spmv_node_fast<4>(sd.m, A, v, a, o32);
    case 14: return spmv_node_fast<14>(sd.m, A, v, a, o32);
    case 5: return spmv_node_fast<5>(sd.m, A, v, a, o32);
    default: return spmv_node_fast<2>(sd.m, A, v, a, o32);
  }
}

// Public apply_wtw.  Every row runs the fast (batched-load, range-mask-only) dot; a row whose
// sum is not finite sets *flag, and apply_wtw then recomputes those rows with
// k_spmv_touched, which multiplies only the pairs the reference's CSR stores (its touched
// pairs, see run_touched): an inf/NaN partner met through an untouched or edge-crossing
// entry (0·inf = NaN here) is skipped there.  Finite rows are exact either way: the skipped
// terms are 0·v with v finite.
template <int SMIN>
__global__ void __launch_bounds__(256) k_spmv(StencilDesc sd, const double* __restrict__ A,
                                              const double* __restrict__ v, double* __restrict__ out,
                                              int* __restrict__ flag, const __grid_constant__ StencilOffsets off) {
  const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= sd.m) return;
  const double acc = spmv_node_fast<SMIN>(sd.m, A, v, a, off.o32);
  if (flag && !isfinite(acc)) *flag = 1;
  out[a] = acc;
}

__global__ void __launch_bounds__(256) k_spmv_touched(StencilDesc sd, const double* __restrict__ A,
                                                      const double* __restrict__ v, const uint8_t* __restrict__ touched,
                                                      double* __restrict__ out,
                                                      const __grid_constant__ StencilOffsets off) {
  const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= sd.m || isfinite(out[a])) return;
  int64_t co[3] = {0, 0, 0};
  int64_t r = a;
#pragma unroll
  for (int k = GSGPC_MAX_DIM - 1; k >= 0; --k) {
    if (k < sd.d) {
      co[k] = r % sd.sz[k];
      r /= sd.sz[k];
    }
  }
  const int64_t m = sd.m;
  double acc = touched[a] ? A[a] * v[a] : 0.0;
  for (int s = 1; s < sd.S_min; ++s) {
    const int64_t o = off.flat[s];
    bool fwd = true, bwd = true;
#pragma unroll
    for (int k = 0; k < GSGPC_MAX_DIM; ++k) {
      if (k < sd.d) {
        const int64_t dk = off.d[s][k];
        fwd = fwd && co[k] + dk >= 0 && co[k] + dk < sd.sz[k];
        bwd = bwd && co[k] - dk >= 0 && co[k] - dk < sd.sz[k];
      }
    }
    if (fwd && touched[s * m + a]) acc = fma(A[s * m + a], v[a + o], acc);
    if (bwd && touched[s * m + a - o]) acc = fma(A[s * m + a - o], v[a - o], acc);
  }
  out[a] = acc;
}

void run_spmv(const Launch& L, const StencilDesc& sd, const double* A, const double* v, double* out, int* flag) {
  const unsigned blocks = static_cast<unsigned>(ceil_div(sd.m, 256));
  const StencilOffsets off = make_stencil_offsets(sd);
  switch (sd.S_min) {
    case 172: k_spmv<172><<<blocks, 256, 0, L.s>>>(sd, A, v, out, flag, off); break;
    case 25: k_spmv<25><<<blocks, 256, 0, L.s>>>(sd, A, v, out, flag, off); break;
    case 4: k_spmv<4><<<blocks, 256, 0, L.s>>>(sd, A, v, out, flag, off); break;
    case 14: k_spmv<14><<<blocks, 256, 0, L.s>>>(sd, A, v, out, flag, off); break;
    case 5: k_spmv<5><<<blocks, 256, 0, L.s>>>(sd, A, v, out, flag, off); break;
    default: k_spmv<2><<<blocks, 256, 0, L.s>>>(sd, A, v, out, flag, off); break;
  }
  L.count();
  GSGPC_CUDA(cudaGetLastError());
}

void run_spmv_touched(const Launch& L, const StencilDesc& sd, const double* A, const double* v,
                      const uint8_t* touched, double* out) {
  k_spmv_touched<<<static_cast<unsigned>(ceil_div(sd.m, 256)), 256, 0, L.s>>>(sd, A, v, touched, out,
                                                                              make_stencil_offsets(sd));
  L.count();
  GSGPC_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ last-block reduction
__device__ __forceinline__ bool arrive_last(unsigned* cnt) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(cnt, 1u);
    last = prev == gridDim.x * gridDim.y - 1;
  }
  __syncthreads();
  return last;
}

template <int NT>
__device__ __forceinline__ double reduce_partials(const double* part, int np, double* sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < np; i += NT) v += part[i];
  return block_sum<NT>(v, sh);
}

// ------------------------------------------------------------------ K4 Toeplitz mode product
struct ToepArgs {
  const double* X;
  double* Y;
  const double* gen;
  int64_t n, inner, outer, L;
  int TL, TA;
};

struct CgEpi {
  const double *r, *u;
  double *s, *z;
  double* part;
  CgState* st;
};

template <int MODE>
__global__ void __launch_bounds__(256) k_toep(ToepArgs t, CgEpi e) {
  extern __shared__ double smem[];
  if (e.st != nullptr && e.st->done) return;
  const int64_t n = t.n;
  double* Ts = smem;
  double* Xs = smem + toep_ts_doubles(n);
  const int64_t l0 = static_cast<int64_t>(blockIdx.x) * t.TL;
  const int nl = static_cast<int>(imin64(t.TL, t.L - l0));
  const int64_t a0 = static_cast<int64_t>(blockIdx.y) * t.TA;
  const int na = static_cast<int>(imin64(t.TA, n - a0));
  toep_load_tile(t.X, t.gen, n, t.inner, t.TL, l0, nl, Ts, Xs, blockDim.x);
  __syncthreads();
  double dot = 0.0;
  const int ngroups = nl * ((na + TOEP_RB - 1) / TOEP_RB);
  for (int uu = threadIdx.x; uu < ngroups; uu += blockDim.x) {
    int tl, ar;
    toep_group(uu, nl, na, t.inner == 1, tl, ar);
    double acc[TOEP_RB];
    toep_dot4(Ts, Xs, n, t.TL, tl, a0 + ar, acc);
    const int64_t l = l0 + tl, o = l / t.inner, i = l % t.inner;
#pragma unroll
    for (int r = 0; r < TOEP_RB; ++r) {
      if (ar + r >= na) break;
      const int64_t g = (o * n + a0 + ar + r) * t.inner + i;
      if (MODE == 0) {
        t.Y[g] = acc[r];
      } else {
        const double beta = e.st->beta;
        const double v = acc[r] + e.st->sigma_sq * e.r[g];
        const double s = e.u[g] + beta * e.s[g];
        const double z = v + beta * e.z[g];
        e.s[g] = s;
        e.z[g] = z;
        dot = fma(s, z, dot);
      }
    }
  }
  if (MODE == 1) {
    __shared__ double sh[8];
    const double bs = block_sum<256>(dot, sh);
    if (threadIdx.x == 0) e.part[blockIdx.y * gridDim.x + blockIdx.x] = bs;
    if (arrive_last(&e.st->cnt_b)) {
      const double pap = reduce_partials<256>(e.part, gridDim.x * gridDim.y, sh);
      if (threadIdx.x == 0) {
        e.st->pap = pap;
        e.st->cnt_b = 0;
      }
    }
  }
}

static void toep_config(int64_t n, int64_t inner, int64_t outer, ToepArgs& t, dim3& grid, size_t& smem) {
  t.n = n;
  t.inner = inner;
  t.outer = outer;
  t.L = inner * outer;
  const int64_t cap = 8192;  // doubles of dynamic smem (64 KB)
  if (toep_smem_doubles(n, 1) > cap) {
    throw Error(GSGPC_UNSUPPORTED, "K_G: grid dimension larger than 2730 nodes is not supported");
  }
  int64_t TL = std::min<int64_t>(32, (cap - toep_ts_doubles(n)) / n);
  TL = std::max<int64_t>(1, std::min<int64_t>(TL, t.L));
  t.TL = static_cast<int>(TL);
  const int64_t tiles = ceil_div(t.L, TL);
  int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(2 * sm_count(), tiles), ceil_div(n, 32)));
  t.TA = static_cast<int>(ceil_div(n, chunks));
  chunks = ceil_div(n, t.TA);
  grid = dim3(static_cast<unsigned>(tiles), static_cast<unsigned>(chunks));
  smem = sizeof(double) * toep_smem_doubles(n, TL);
}

static void launch_toep(const Launch& L, int mode, ToepArgs t, dim3 grid, size_t smem, CgEpi e) {
  if (mode == 0) {
    if (smem > 48 * 1024) set_max_dynamic_smem(reinterpret_cast<const void*>(k_toep<0>), 64 * 1024);
    k_toep<0><<<grid, 256, smem, L.s>>>(t, e);
  } else {
    if (smem > 48 * 1024) set_max_dynamic_smem(reinterpret_cast<const void*>(k_toep<1>), 64 * 1024);
    k_toep<1><<<grid, 256, smem, L.s>>>(t, e);
  }
  L.count();
  GSGPC_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ K4' Toeplitz mode by FFT
// Dimensions too long for the shared-memory / tensor-core mode products (the reference takes
// any grid): the product with T_k runs as the reference's circulant embedding
// (grid.cpp:94-151, 193-235) restricted to one factor of the separable SE kernel — every line
// along k is zero-padded to e_k = next_fast_fft_size(2 n_k − 1), transformed (batched r2c,
// cuFFT), multiplied by the spectrum of T_k's embedded first column, transformed back (c2r)
// and scaled by 1/e_k.  O(m log e_k) per mode instead of O(m n_k).
int64_t next_fast_fft_size(int64_t x) {
  if (x < 1) return 1;
  for (int64_t n = x;; ++n) {
    int64_t r = n;
    while (r % 2 == 0) r /= 2;
    while (r % 3 == 0) r /= 3;
    while (r % 5 == 0) r /= 5;
    if (r == 1) return n;
  }
}

#define GSGPC_CUFFT(expr)                                                                          \
  do {                                                                                             \
    const cufftResult _r = (expr);                                                                 \
    if (_r != CUFFT_SUCCESS)                                                                       \
      throw ::gsgpc::Error(GSGPC_CUDA_ERROR, std::string(#expr " failed: cufftResult ") + std::to_string(_r)); \
  } while (0)

struct KgFft {
  int d = 0;
  int device = 0;
  bool on[GSGPC_MAX_DIM] = {};
  int64_t n[GSGPC_MAX_DIM] = {}, e[GSGPC_MAX_DIM] = {};
  double2* spec[GSGPC_MAX_DIM] = {};
  std::map<std::pair<int, int64_t>, std::pair<cufftHandle, cufftHandle>> plans;  // (dim, lines) → r2c, c2r
  double* rbuf = nullptr;
  double2* cbuf = nullptr;
  size_t rcap = 0, ccap = 0;
  std::mutex mu;
  ~KgFft() {
    cudaSetDevice(device);
    for (auto& kv : plans) {
      cufftDestroy(kv.second.first);
      cufftDestroy(kv.second.second);
    }
    for (auto* p : spec) cudaFree(p);
    cudaFree(rbuf);
    cudaFree(cbuf);
  }
  // plans + scratch for `lines` lines of dimension k (not inside a stream capture)
  std::pair<cufftHandle, cufftHandle> plan(int k, int64_t lines) {
    auto it = plans.find({k, lines});
    if (it != plans.end()) return it->second;
    const size_t need_r = static_cast<size_t>(lines) * e[k], need_c = static_cast<size_t>(lines) * (e[k] / 2 + 1);
    if (need_r > rcap) {
      cudaFree(rbuf);
      rbuf = nullptr;
      GSGPC_CUDA(cudaMalloc(&rbuf, sizeof(double) * need_r));
      rcap = need_r;
    }
    if (need_c > ccap) {
      cudaFree(cbuf);
      cbuf = nullptr;
      GSGPC_CUDA(cudaMalloc(&cbuf, sizeof(double2) * need_c));
      ccap = need_c;
    }
    int nn = static_cast<int>(e[k]);
    const int hc = static_cast<int>(e[k] / 2 + 1);
    cufftHandle f, b;
    GSGPC_CUFFT(cufftPlanMany(&f, 1, &nn, nullptr, 1, nn, nullptr, 1, hc, CUFFT_D2Z, static_cast<int>(lines)));
    GSGPC_CUFFT(cufftPlanMany(&b, 1, &nn, nullptr, 1, hc, nullptr, 1, nn, CUFFT_Z2D, static_cast<int>(lines)));
    plans[{k, lines}] = {f, b};
    return {f, b};
  }
};

bool kg_fft_dim(const KgDev& kg, int k) { return kg.fft != nullptr && kg.fft->on[k]; }

// circulant embedding of a symmetric Toeplitz column: c[j] = g[δ(j)], δ = j (j < n),
// e − j (e − j < n), else none (grid.cpp:120-138)
__global__ void k_fft_embed_gen(const double* __restrict__ gen, int64_t n, int64_t e, double* __restrict__ c) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= e) return;
  c[j] = j < n ? gen[j] : (e - j < n ? gen[e - j] : 0.0);
}

// lines of X ([outer][n][inner]) → zero-padded rows rb[l][0..e), l = o·inner + i
__global__ void k_fft_scatter(const double* __restrict__ X, int64_t n, int64_t inner, int64_t lines, int64_t e,
                              double* __restrict__ rb, const CgState* st) {
  if (st != nullptr && st->done) return;
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= lines * e) return;
  const int64_t l = q / e, j = q - l * e;
  const int64_t o = l / inner, i = l - o * inner;
  rb[q] = j < n ? X[(o * n + j) * inner + i] : 0.0;
}

__global__ void k_fft_mul(double2* __restrict__ cb, const double2* __restrict__ spec, int64_t hc, int64_t total,
                          const CgState* st) {
  if (st != nullptr && st->done) return;
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= total) return;
  const double2 a = cb[q], b = spec[q % hc];
  cb[q] = make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// rb[l][a] / e → Y in [outer][n][inner] order; MODE 1: the CG epilogue of k_toep
template <int MODE>
__global__ void __launch_bounds__(256) k_fft_gather(const double* __restrict__ rb, int64_t n, int64_t inner,
                                                    int64_t total, int64_t e, double scale, double* __restrict__ Y,
                                                    CgEpi ep) {
  if (ep.st != nullptr && ep.st->done) return;
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double dot = 0.0;
  if (g < total) {
    const int64_t i = g % inner, t = g / inner, a = t % n, o = t / n;
    const double acc = rb[(o * inner + i) * e + a] * scale;
    if (MODE == 0) {
      Y[g] = acc;
    } else {
      const double beta = ep.st->beta;
      const double v = acc + ep.st->sigma_sq * ep.r[g];
      const double s = ep.u[g] + beta * ep.s[g];
      const double z = v + beta * ep.z[g];
      ep.s[g] = s;
      ep.z[g] = z;
      dot = s * z;
    }
  }
  if (MODE == 1) {
    __shared__ double sh[8];
    const double bs = block_sum<256>(dot, sh);
    if (threadIdx.x == 0) ep.part[blockIdx.x] = bs;
    if (arrive_last(&ep.st->cnt_b)) {
      const double pap = reduce_partials<256>(ep.part, gridDim.x, sh);
      if (threadIdx.x == 0) {
        ep.st->pap = pap;
        ep.st->cnt_b = 0;
      }
    }
  }
}

std::shared_ptr<KgFft> kg_fft_create(const KgDev& kg, int64_t min_nodes, cudaStream_t s) {
  bool any = false;
  for (int k = 0; k < kg.d; ++k) any = any || kg.sz[k] >= min_nodes;
  if (!any) return nullptr;
  auto f = std::make_shared<KgFft>();
  f->d = kg.d;
  GSGPC_CUDA(cudaGetDevice(&f->device));
  for (int k = 0; k < kg.d; ++k) {
    if (kg.sz[k] < min_nodes) continue;
    f->on[k] = true;
    f->n[k] = kg.sz[k];
    f->e[k] = next_fast_fft_size(2 * kg.sz[k] - 1);
    const int64_t e = f->e[k], hc = e / 2 + 1;
    GSGPC_CUDA(cudaMalloc(&f->spec[k], sizeof(double2) * hc));
    double* col = nullptr;
    GSGPC_CUDA(cudaMalloc(&col, sizeof(double) * e));
    k_fft_embed_gen<<<static_cast<unsigned>(ceil_div(e, 256)), 256, 0, s>>>(kg.gen[k], kg.sz[k], e, col);
    cufftHandle p;
    int nn = static_cast<int>(e);
    GSGPC_CUFFT(cufftPlan1d(&p, nn, CUFFT_D2Z, 1));
    GSGPC_CUFFT(cufftSetStream(p, s));
    GSGPC_CUFFT(cufftExecD2Z(p, col, f->spec[k]));
    GSGPC_CUDA(cudaStreamSynchronize(s));
    cufftDestroy(p);
    cudaFree(col);
    f->plan(k, kg.m / kg.sz[k]);  // one m-vector (the solvers' case; ready before any graph capture)
  }
  GSGPC_CUDA(cudaGetLastError());
  return f;
}

static void fft_mode(const Launch& L, KgFft& f, int k, const double* X, double* Y, int64_t inner, int64_t outer,
                     int mode, CgEpi e) {
  std::lock_guard<std::mutex> lk(f.mu);
  const int64_t n = f.n[k], E = f.e[k], hc = E / 2 + 1, lines = inner * outer;
  const auto pl = f.plan(k, lines);
  const CgState* st = e.st;
  k_fft_scatter<<<static_cast<unsigned>(ceil_div(lines * E, 256)), 256, 0, L.s>>>(X, n, inner, lines, E, f.rbuf, st);
  GSGPC_CUFFT(cufftSetStream(pl.first, L.s));
  GSGPC_CUFFT(cufftExecD2Z(pl.first, f.rbuf, f.cbuf));
  k_fft_mul<<<static_cast<unsigned>(ceil_div(lines * hc, 256)), 256, 0, L.s>>>(f.cbuf, f.spec[k], hc, lines * hc, st);
  GSGPC_CUFFT(cufftSetStream(pl.second, L.s));
  GSGPC_CUFFT(cufftExecZ2D(pl.second, f.cbuf, f.rbuf));
  const int64_t total = lines * n;
  const unsigned gb = static_cast<unsigned>(ceil_div(total, 256));
  if (mode == 0) k_fft_gather<0><<<gb, 256, 0, L.s>>>(f.rbuf, n, inner, total, E, 1.0 / static_cast<double>(E), Y, e);
  else k_fft_gather<1><<<gb, 256, 0, L.s>>>(f.rbuf, n, inner, total, E, 1.0 / static_cast<double>(E), Y, e);
  L.count(3);
  GSGPC_CUDA(cudaGetLastError());
}

// Applies T_{d-1}, ..., T_1 (plain) and T_0 (MODE, possibly with the CG epilogue).
// batch > 1: `batch` contiguous m-vectors, the batch index an extra outermost dimension.
static void kg_chain(const Launch& L, const KgDev& kg, const double* v, double* out, double* tmp0, double* tmp1,
                     int last_mode, CgEpi e, int64_t batch = 1) {
  const double* cur = v;
  for (int k = kg.d - 1; k >= 0; --k) {
    int64_t inner = 1, outer = batch;
    for (int j = k + 1; j < kg.d; ++j) inner *= kg.sz[j];
    for (int j = 0; j < k; ++j) outer *= kg.sz[j];
    double* dst = k == 0 ? out : (cur == tmp0 ? tmp1 : tmp0);
    if (kg_fft_dim(kg, k)) {
      fft_mode(L, *kg.fft, k, cur, dst, inner, outer, k == 0 ? last_mode : 0, e);
      cur = dst;
      continue;
    }
    ToepArgs t{};
    dim3 grid;
    size_t smem;
    toep_config(kg.sz[k], inner, outer, t, grid, smem);
    t.X = cur;
    t.gen = kg.gen[k];
    t.Y = dst;
    launch_toep(L, k == 0 ? last_mode : 0, t, grid, smem, e);
    cur = dst;
  }
}

void run_kg_apply(const Launch& L, const KgDev& kg, const double* v, double* out, double* tmp0, double* tmp1) {
  CgEpi e{};
  kg_chain(L, kg, v, out, tmp0, tmp1, 0, e);
}

void run_kg_apply_batched(const Launch& L, const KgDev& kg, int64_t batch, const double* v, double* out,
                          double* tmp0, double* tmp1) {
  CgEpi e{};
  kg_chain(L, kg, v, out, tmp0, tmp1, 0, e, batch);
}

int cg_partials_needed(int64_t m) {
  return static_cast<int>(std::max<int64_t>(ceil_div(m, 256), 4096));
}

// ------------------------------------------------------------------ K5 EFCG kernels
__global__ void __launch_bounds__(256) k_cg_update(CgBufs b, int64_t m) {
  CgState* st = b.st;
  if (st->done) return;
  if (st->iter >= st->maxiter) {
    if (blockIdx.x == 0 && threadIdx.x == 0) st->done = 1;
    return;
  }
  const double pap = st->pap;
  if (pap <= 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->breakdown = 1;
      st->done = 1;
    }
    return;
  }
  const double alpha = st->rho / pap;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < m) {
    b.x[i] += alpha * b.s[i];
    b.r[i] -= alpha * b.z[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->alpha = alpha;
    b.alphas[st->iter] = alpha;
  }
}

template <int INIT>
__global__ void __launch_bounds__(256) k_cg_spmv(StencilDesc sd, const double* __restrict__ A, CgBufs b,
                                                 const __grid_constant__ StencilOffsets off) {
  CgState* st = b.st;
  if (st->done) return;
  __shared__ double sh[8];
  const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double d = 0.0;
  if (a < sd.m) {
    const double u = spmv_node_any(sd, A, b.r, a, off.o32);
    b.u[a] = u;
    d = u * b.r[a];
  }
  const double bs = block_sum<256>(d, sh);
  if (threadIdx.x == 0) b.part_a[blockIdx.x] = bs;
  if (arrive_last(&st->cnt_a)) {
    const double rho_new = reduce_partials<256>(b.part_a, gridDim.x, sh);
    if (threadIdx.x == 0) {
      st->cnt_a = 0;
      if (INIT) {
        st->rho = rho_new;
        st->eps = st->eps_abs >= 0.0 ? st->eps_abs : st->rel_tol * st->rel_tol * rho_new;
        b.trace[0] = rho_new;
        st->beta = 0.0;
        if (rho_new <= st->eps) {
          st->converged = 1;
          st->done = 1;
        }
      } else {
        st->iter += 1;
        b.trace[st->iter] = rho_new;
        if (rho_new <= st->eps) {
          st->converged = 1;
          st->done = 1;
          st->rho = rho_new;
        } else {
          const double beta = rho_new / st->rho;
          st->beta = beta;
          b.betas[st->iter - 1] = beta;
          st->rho = rho_new;
        }
      }
    }
  }
}

void run_cg_init(const Launch& L, const StencilDesc& sd, const double* A, const KgDev& kg, const CgBufs& b,
                 int64_t m) {
  k_cg_spmv<1><<<static_cast<unsigned>(ceil_div(m, 256)), 256, 0, L.s>>>(sd, A, b, make_stencil_offsets(sd));
  L.count();
  CgEpi e{b.r, b.u, b.s, b.z, b.part_b, b.st};
  kg_chain(L, kg, b.u, nullptr, b.kt0, b.kt1, 1, e);
  GSGPC_CUDA(cudaGetLastError());
}

void run_cg_iter(const Launch& L, const StencilDesc& sd, const double* A, const KgDev& kg, const CgBufs& b,
                 int64_t m) {
  k_cg_update<<<static_cast<unsigned>(ceil_div(m, 256)), 256, 0, L.s>>>(b, m);
  k_cg_spmv<0><<<static_cast<unsigned>(ceil_div(m, 256)), 256, 0, L.s>>>(sd, A, b, make_stencil_offsets(sd));
  L.count(2);
  CgEpi e{b.r, b.u, b.s, b.z, b.part_b, b.st};
  kg_chain(L, kg, b.u, nullptr, b.kt0, b.kt1, 1, e);
  GSGPC_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ vector helpers
__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b, const double* __restrict__ y,
                        double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a * x[i] + b * y[i];
}
// out = x + y / b (the reference's  x̂_d + W^T y / σ²  and  -K w / σ²  forms: division, not
// multiplication by the reciprocal)
__global__ void k_add_div(int64_t n, const double* __restrict__ x, const double* __restrict__ y, double b, double sx,
                          double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (x ? sx * x[i] : 0.0) + y[i] / b;
}

void run_axpby(const Launch& L, int64_t n, double a, const double* x, double b, const double* y, double* out) {
  k_axpby<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, L.s>>>(n, a, x, b, y, out);
  L.count();
  GSGPC_CUDA(cudaGetLastError());
}

void run_add_div(const Launch& L, int64_t n, const double* x, double sx, const double* y, double b, double* out) {
  k_add_div<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, L.s>>>(n, x, y, b, sx, out);
  L.count();
  GSGPC_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ pointwise interpolation
// interp_weights (interp.cpp:79-134), bit-exact, one thread per point.
template <typename T, bool PREDICT>
__global__ void __launch_bounds__(128) k_interp(PointsDev p, int64_t n, GridDev g, int64_t* __restrict__ idx,
                                                double* __restrict__ w, int* __restrict__ nnz,
                                                int* __restrict__ status, const double* __restrict__ coeffs,
                                                double* __restrict__ pred) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x[GSGPC_MAX_DIM], y;
  const T* X = static_cast<const T*>(p.x);
#pragma unroll
  for (int k = 0; k < GSGPC_MAX_DIM; ++k) x[k] = k < g.d ? static_cast<double>(X[i * p.xs + p.xo[k]]) : 0.0;
  (void)y;
  int64_t st0[GSGPC_MAX_DIM];
  double wk[GSGPC_MAX_DIM][4];
  int stt = PT_VALID;
  for (int k = 0; k < g.d; ++k) {
    int64_t i0 = 0;
    double t = 0.0;
    const int s = stencil_dim(x[k], g.mn[k], g.sp[k], g.sz[k], i0, t);
    if (s == PT_OUTSIDE) {
      stt = PT_OUTSIDE;
      break;
    }
    if (s == PT_EMPTY) {
      // NaN: the reference's floor()/cast yields an index whose weights are all zero
      for (int o = 0; o < 4; ++o) wk[k][o] = 0.0;
      st0[k] = 0;
      continue;
    }
    weights_1d(t, g.W, wk[k]);
    st0[k] = g.W == 4 ? i0 - 1 : i0;
  }
  int cnt = 0;
  double out = 0.0;
  const int width = g.W;
  const int64_t cap = PREDICT ? 0 : 1;
  (void)cap;
  if (stt == PT_VALID) {
    int combos = 1;
    for (int k = 0; k < g.d; ++k) combos *= width;
    const int64_t rowcap = combos;
    for (int c = 0; c < combos; ++c) {
      int offs[GSGPC_MAX_DIM];
      int cc = c;
      for (int k = g.d - 1; k >= 0; --k) {
        offs[k] = cc % width;
        cc /= width;
      }
      double wv = 1.0;
      int64_t flat = 0;
      bool in_range = true;
      for (int k = 0; k < g.d; ++k) {
        const double wkk = wk[k][offs[k]];
        if (wkk == 0.0) {
          wv = 0.0;
          break;
        }
        const int64_t j = st0[k] + offs[k];
        if (j < 0 || j >= g.sz[k]) {
          in_range = false;
          break;
        }
        wv = __dmul_rn(wv, wkk);
        flat = flat * g.sz[k] + j;
      }
      if (wv != 0.0) {
        if (!in_range) {
          stt = PT_LEAVES;
          break;
        }
        if (PREDICT) {
          out = __dadd_rn(out, __dmul_rn(wv, coeffs[flat]));
        } else {
          idx[i * rowcap + cnt] = flat;
          w[i * rowcap + cnt] = wv;
        }
        ++cnt;
      }
    }
  }
  if (stt != PT_VALID) cnt = 0;
  if (PREDICT) {
    pred[i] = stt == PT_VALID ? out : 0.0;
    if (status) status[i] = stt == PT_VALID ? 0 : stt;
  } else {
    nnz[i] = cnt;
    status[i] = stt == PT_VALID ? 0 : stt;
  }
}

void run_interp_weights(const Launch& L, int dtype, const PointsDev& p, int64_t n, const GridDev& g, int64_t* idx,
                        double* w, int* nnz, int* status) {
  const unsigned blocks = static_cast<unsigned>(ceil_div(n, 128));
  if (dtype == GSGPC_F32) k_interp<float, false><<<blocks, 128, 0, L.s>>>(p, n, g, idx, w, nnz, status, nullptr, nullptr);
  else k_interp<double, false><<<blocks, 128, 0, L.s>>>(p, n, g, idx, w, nnz, status, nullptr, nullptr);
  L.count();
  GSGPC_CUDA(cudaGetLastError());
}

void run_predict(const Launch& L, int dtype, const PointsDev& p, int64_t n, const GridDev& g, const double* coeffs,
                 double* out, int* status) {
  const unsigned blocks = static_cast<unsigned>(ceil_div(n, 128));
  if (dtype == GSGPC_F32) k_interp<float, true><<<blocks, 128, 0, L.s>>>(p, n, g, nullptr, nullptr, nullptr, status, coeffs, out);
  else k_interp<double, true><<<blocks, 128, 0, L.s>>>(p, n, g, nullptr, nullptr, nullptr, status, coeffs, out);
  L.count();
  GSGPC_CUDA(cudaGetLastError());
}

}  // namespace gsgpc
