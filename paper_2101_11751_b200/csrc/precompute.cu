// precompute.cu — the O(n) sufficient-statistics pass (replaces
// SufficientStatsAccumulator::add/finalize + sufficient_stats, interp.cpp:179-263).
//
// Pipeline per batch of rows (all on one stream):
//   K2a  k_classify_count : stencil_1d for every point (bit-exact), error row (atomicMin),
//                           per-cell histogram (warp-aggregated atomics), Σy² partials.
//   K2b  scan             : exclusive scan of the histogram → cell offsets.
//   K2c  k_scatter        : counting-sort scatter of the raw rows by cell.
//   K1   k_moments_*      : per-cell polynomial moments  M_c[e] = Σ_p Π_k t_pk^{e_k}
//                           (e_k ≤ 2W-2) and  Y_c[e] = Σ_p y_p Π_k t_pk^{e_k} (e_k ≤ W-1),
//                           accumulated in registers over the points of one cell, flushed
//                           once per (warp range, cell) — RMW when the warp owns the cell,
//                           REDG otherwise.  Probe images use the same pass (k_probe_moments).
// finalize (on demand): cell-major moments → moment-major (transpose), then one separable
//   transform per dimension maps (cell, exponent) → (node, stencil offset) with the fixed
//   product-polynomial coefficients of the Keys / linear weights, giving the W^T W stencil
//   (symmetric half, offset-major) and W^T y.  Exact because every 1-D weight is a
//   polynomial of degree W-1 in the in-cell offset t ∈ [0,1].
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "internal.cuh"
#include "precompute.cuh"

namespace gsgpc {

bool debug_sync_enabled() {
  static const bool on = getenv("GSGPC_DEBUG_SYNC") != nullptr;
  return on;
}

void debug_sync_check(cudaStream_t s, uint64_t ordinal) {
  const cudaError_t e = cudaStreamSynchronize(s);
  const cudaError_t l = cudaGetLastError();
  if (e != cudaSuccess || l != cudaSuccess) {
    fprintf(stderr, "[gsgpc debug] launch #%llu failed: %s\n", static_cast<unsigned long long>(ordinal),
            cudaGetErrorString(e != cudaSuccess ? e : l));
    throw Error(GSGPC_CUDA_ERROR, std::string("launch #") + std::to_string(ordinal) + " failed: " +
                                      cudaGetErrorString(e != cudaSuccess ? e : l));
  }
}

// Polynomial form of the 1-D weights on t ∈ [0,1] (expanded from interp.cpp:27-37 on the
// branch each stencil slot takes): cubic slots c(t+1), c(t), c(1-t), c(2-t); linear
// slots l(t), l(1-t).  All coefficients are dyadic, so the tables are exact in fp64.
// Both schemes' tables are compile-time constants (no per-call upload, so contexts and
// threads using different schemes on one device never see each other's tables).
struct PolyTables {
  double C[4 * 4 * 7];  // C[i][j][e]: coefficient of t^e in w_i(t) w_j(t)
  double P[4 * 4];      // P[i][e]: coefficient of t^e in w_i(t)
};

constexpr PolyTables make_poly_tables(int W) {
  PolyTables t{};
  if (W == 4) {
    const double p[4][4] = {{0.0, -0.5, 1.0, -0.5},
                            {1.0, 0.0, -2.5, 1.5},
                            {0.0, 0.5, 2.0, -1.5},
                            {0.0, 0.0, -0.5, 0.5}};
    for (int i = 0; i < 4; ++i)
      for (int e = 0; e < 4; ++e) t.P[i * 4 + e] = p[i][e];
  } else {
    t.P[0 * 4 + 0] = 1.0;
    t.P[0 * 4 + 1] = -1.0;
    t.P[1 * 4 + 1] = 1.0;
  }
  for (int i = 0; i < W; ++i)
    for (int j = 0; j < W; ++j)
      for (int a = 0; a < W; ++a)
        for (int b = 0; b < W; ++b) t.C[(i * 4 + j) * 7 + a + b] += t.P[i * 4 + a] * t.P[j * 4 + b];
  return t;
}

__constant__ PolyTables c_poly[2] = {make_poly_tables(2), make_poly_tables(4)};  // [0] linear, [1] cubic

// ------------------------------------------------------------------ K2a classify + count
// classify() specialised on the dimension, branch-light, 32-bit cell arithmetic
// (cells < 2^31).  Same decisions as the reference (see stencil_dim_fast for the snap
// argument).  Non-snapped offsets satisfy t ∈ [1e-9, 1 - 1e-9], where every Keys slot is
// nonzero (the pieces vanish only at integer arguments), so "stencil leaves the grid" is
// exactly (i0 == 0 || i0 + 2 >= size) && t ∉ {0, 1} for cubic and never for linear.
// Rows whose |u - round(u)| lies within a few ulp of the 1e-9 snap tolerance take the
// exact-division path.
// Exact (division) path for the rare rows near the snap tolerance; coordinates by value and
// (status, cell) packed in the return value so the never-taken call forces nothing to the stack.
template <int D>
__device__ __noinline__ long long classify_exact(const GridDev& g, double x0, double x1, double x2) {
  int64_t i0[GSGPC_MAX_DIM];
  double t[GSGPC_MAX_DIM];
  double xx[GSGPC_MAX_DIM] = {x0, x1, x2};
  int64_t c = 0;
  GridDev gd = g;
  gd.d = D;
  const int st = classify(gd, xx, i0, t, c);
  return (static_cast<long long>(st) << 32) | static_cast<unsigned>(c);
}

template <int D>
__device__ __forceinline__ int classify_d(const GridDev& g, const double* x, int& cell) {
  double u[D];
  bool band = false;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const double uu = __dsub_rn(x[k], g.mn[k]) * g.isp[k];
    const double r = rint(uu);
    const double dd = fabs(uu - r);
    const double e = 1e-12 + fabs(uu) * 3.552713678800501e-15;
    band = band || fabs(dd - 1e-9) <= e;  // dd within e of the snap tolerance
    u[k] = dd < 1e-9 ? r : uu;
  }
  if (band) {
    const long long pk = classify_exact<D>(g, x[0], D > 1 ? x[1] : 0.0, D > 2 ? x[2] : 0.0);
    cell = static_cast<int>(static_cast<unsigned>(pk));
    return static_cast<int>(pk >> 32);
  }
  bool outside = false;
#pragma unroll
  for (int k = 0; k < D; ++k) outside = outside || u[k] < 0.0 || u[k] > static_cast<double>(g.sz[k] - 1);
  if (outside) return PT_OUTSIDE;
  int c = 0, st = PT_VALID;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const bool isnan_k = u[k] != u[k];
    const int sz = static_cast<int>(g.sz[k]);
    int i0 = isnan_k ? 0 : __double2int_rd(u[k]);
    i0 = min(i0, sz - 2);
    const double t = u[k] - static_cast<double>(i0);
    const bool leaves = g.W == 4 && (i0 == 0 || i0 + 2 >= sz) && t != 0.0 && t != 1.0;
    if (st == PT_VALID) st = isnan_k ? PT_EMPTY : (leaves ? PT_LEAVES : PT_VALID);
    c = c * static_cast<int>(g.nc[k]) + i0;
  }
  cell = c;
  return st;
}

// Rows are processed UNR at a time per thread (all loads issued before any use) so each
// warp keeps UNR row loads — and, in the scatter, UNR atomics and stores — in flight.
constexpr int SORT_UNR = 8;

template <typename T, bool PACKED>
__device__ __forceinline__ void load_row(const PointsDev& p, int d, int64_t i, T* v) {
  if (PACKED) {
    // (x0, x1, x2, y) rows, 4·sizeof(T)-aligned
    if (sizeof(T) == 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(p.x) + i);
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
      const double2 a = __ldg(reinterpret_cast<const double2*>(p.x) + 2 * i);
      const double2 b = __ldg(reinterpret_cast<const double2*>(p.x) + 2 * i + 1);
      v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
  } else {
    const T* X = static_cast<const T*>(p.x);
    const T* Y = static_cast<const T*>(p.y);
#pragma unroll
    for (int k = 0; k < 3; ++k) v[k] = k < d ? X[i * p.xs + p.xo[k]] : T(0);
    v[3] = Y[i * p.ys];
  }
}

// ------------------------------------------------------------------ device gate
// The binning → moments chain of a batch runs without a host round trip: kernels are sized
// by host upper bounds (rows of the batch) and read the true counts (rows binned, slices)
// from the device; every kernel that commits to the accumulator returns at once when the
// classify pass recorded an out-of-grid row (the host checks that word once per call, after
// the work, and throws — nothing was committed).
struct BinGate {
  const unsigned long long* err;  // ~0: no error
  const int64_t* rows_end;        // rows binned (bbase[nb]); nullptr → the host value
  __device__ __forceinline__ bool closed() const { return err != nullptr && *err != ~0ull; }
  __device__ __forceinline__ int64_t rows(int64_t host_value) const {
    return rows_end != nullptr ? min(host_value, *rows_end) : host_value;
  }
};

// ------------------------------------------------------------------ deterministic ranks
// The counting sorts of the binning hand out slots from shared-memory atomicAdd cursors in
// arrival order, so the rows of a cell reached K1 — and the fp64 sums — in a different order
// every run.  Deterministic ranks without per-item block barriers:
//   1. warp_rank: each warp ranks its own items per key against its own row of a per-warp
//      count table (u16, nkeys per warp): the lanes holding the same key (one ballot per key
//      bit — MATCH.ANY, a long MIO operation, stalled the partition and slice scatters on
//      its result) give the rank inside a round, the row the warp's earlier rounds;
//   2. after one block barrier, col_prefix turns every key's column into the exclusive prefix
//      over the warps and returns the key's total.
// An item's slot = key start + prefix[warp][key] + rank: order (warp, round, lane), fixed.
constexpr int BIN_MAX_BSH = 14;  // bucket-sort shared counters: 2^14 ints (keys of ≤ 14 bits)
constexpr int64_t BIN_MAX_NB = 8192;  // buckets: k_tscan_buckets handles 8 per thread

// lanes whose key equals this lane's (keys < 2^nbits, or −1): nbits + 1 ballots
__device__ __forceinline__ unsigned warp_peers(int key, int nbits) {
  const bool valid = key >= 0;
  const unsigned v = __ballot_sync(0xffffffffu, valid);
  unsigned peers = valid ? v : ~v;
#pragma unroll 1
  for (int b = 0; b < BIN_MAX_BSH; ++b) {
    if (b < nbits) {  // warp-uniform
      const bool bit = (key >> b) & 1;
      const unsigned m = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? m : ~m;
    }
  }
  return peers;
}

// nbits < 0: the peers from MATCH.ANY instead of ballots
__device__ __forceinline__ int warp_rank(int key, int nbits, uint16_t* __restrict__ row) {
  const int lane = threadIdx.x & 31;
  const unsigned peers = nbits < 0 ? __match_any_sync(0xffffffffu, key) : warp_peers(key, nbits);
  const int leader = __ffs(peers) - 1;
  int base = 0;
  if (key >= 0 && lane == leader) {
    base = row[key];
    row[key] = static_cast<uint16_t>(base + __popc(peers));
  }
  base = __shfl_sync(0xffffffffu, base, leader);
  __syncwarp();
  return key >= 0 ? base + __popc(peers & ((1u << lane) - 1u)) : -1;
}

// column key of the [NW][nkeys] table → exclusive prefix over warps (+ add), returns the total
template <int NW>
__device__ __forceinline__ int col_prefix(uint16_t* __restrict__ tab, int nkeys, int key, int add) {
  int run = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int v = tab[w * nkeys + key];
    tab[w * nkeys + key] = static_cast<uint16_t>(run + add);
    run += v;
  }
  return run;
}

// ------------------------------------------------------------------ K2 binning
// Two-level counting sort, no per-row global atomics.  Rows are cut into tiles of
// TILE_ROWS; cells into buckets of 2^bsh consecutive (row-major) cells, nb ≤ ~1024 buckets.
//   K2a classify : exact cell of every row → cellid[i] (-1: not interpolated); per-tile
//                  bucket histogram from shared-memory atomics → tcnt[tile][bucket]; error
//                  row (atomicMin); Σy² partials.
//   K2b totals   : bucket sizes → bbase (row offsets), sbase (slice offsets).
//   K2c partition: each tile claims one run per bucket from the bucket's cursor and writes
//                  its rows there (shared-memory cursors) → bucket-contiguous rows + cell ids.
//   K2d slices   : per-bucket counting sort by cell in SLICE_ROWS slices (count, scan,
//                  scatter with shared-memory cursors) → cell-sorted rows, off[cells + 1].
// A direct counting sort (one global cursor atomic per row on 1.3e5 hot counters) was
// latency-bound at ~1.7 TB/s; this pays one extra pass over the rows for no per-row global
// atomics and at most nb + slices write frontiers.
template <typename T>
struct alignas(sizeof(T) * 4) Row4 {
  T v[4];  // x0, x1, x2 (unused dims 0), y
};

__device__ __forceinline__ float ld_l2_64(const float* p) {
  float v;
  asm volatile("ld.global.nc.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_l2_64(const double* p) {
  double v;
  asm volatile("ld.global.nc.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// The rows of a batch in cell order, as K1 reads them: sorted row index p → the row gathered
// from the caller's layout (one vector load for packed (x0, x1, x2, y) rows).  The binning
// sorts 4-byte indices only; K1 is FP64-bound at d = 3, so the gathers' latency hides under
// the MMAs (each batch's rows are requested one batch ahead).
template <typename T, bool PACKED>
struct RowSrc {
  PointsDev pts;
  const int* __restrict__ idx;  // sorted row → batch row
  int d;
  __device__ __forceinline__ int64_t at(int64_t p) const { return __ldg(idx + p); }
  // by batch row index.  The gathers are random over the whole input: each asks L2 for 64-byte
  // fills (.L2::64B) instead of the default 128 (config 3 K1: 15.5 → 8.4 GB of DRAM reads per
  // launch), packed rows without allocating in L1.
  __device__ __forceinline__ Row4<T> row(int64_t i) const {
    Row4<T> r;
    if (PACKED && sizeof(T) == 4) {
      float4 q;
      asm volatile("ld.global.L1::no_allocate.L2::64B.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w)
                   : "l"(reinterpret_cast<const float4*>(pts.x) + i));
      r.v[0] = q.x; r.v[1] = q.y; r.v[2] = q.z; r.v[3] = q.w;
    } else if (PACKED) {
      const double* p = static_cast<const double*>(pts.x) + 4 * i;
      double a0, a1, b0, b1;
      asm volatile("ld.global.L1::no_allocate.L2::64B.v2.f64 {%0,%1}, [%2];" : "=d"(a0), "=d"(a1) : "l"(p));
      asm volatile("ld.global.L1::no_allocate.L2::64B.v2.f64 {%0,%1}, [%2];" : "=d"(b0), "=d"(b1) : "l"(p + 2));
      r.v[0] = static_cast<T>(a0); r.v[1] = static_cast<T>(a1); r.v[2] = static_cast<T>(b0); r.v[3] = static_cast<T>(b1);
    } else {
      const T* X = static_cast<const T*>(pts.x);
      const T* Y = static_cast<const T*>(pts.y);
#pragma unroll
      for (int k = 0; k < 3; ++k) r.v[k] = k < d ? ld_l2_64(X + i * pts.xs + pts.xo[k]) : T(0);
      r.v[3] = ld_l2_64(Y + i * pts.ys);
    }
    return r;
  }
  __device__ __forceinline__ Row4<T> operator[](int64_t p) const { return row(at(p)); }
};

constexpr int TILE_ROWS = 32768;  // classify tile (bucket histogram): 256 threads × SORT_UNR × 16
// Build-time knobs (B200, config 3, partition + slice sort = 2.20 ms with the defaults):
// 512-thread partition blocks ×2 per SM 2.32 ms.
#ifndef PART_NT_DEF
#define PART_NT_DEF 512
#endif
#ifndef PART_MINB
#define PART_MINB 2
#endif
constexpr int PART_NT = PART_NT_DEF;  // partition: PART_MINB blocks of PART_NT threads per SM

template <typename T, bool PACKED, int D>
__global__ void __launch_bounds__(256, 3) k_classify_tiles(PointsDev pts, int64_t n, int64_t row0, GridDev g,
                                                         int bsh, int nb, int* __restrict__ tcnt,
                                                         unsigned long long* __restrict__ err,
                                                         double* __restrict__ yty_part,
                                                         int* __restrict__ cellid) {
  extern __shared__ int hist[];
  __shared__ double sh[8];
  double ysq = 0.0;
  const int64_t ntiles = (n + TILE_ROWS - 1) / TILE_ROWS;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    for (int j = threadIdx.x; j < nb; j += blockDim.x) hist[j] = 0;
    __syncthreads();
    for (int sub = 0; sub < TILE_ROWS / (256 * SORT_UNR); ++sub) {
      const int64_t base = tile * TILE_ROWS + static_cast<int64_t>(sub) * 256 * SORT_UNR;
      T v[SORT_UNR][4];
#pragma unroll
      for (int u = 0; u < SORT_UNR; ++u) {
        const int64_t i = base + threadIdx.x + static_cast<int64_t>(u) * 256;
        if (i < n) load_row<T, PACKED>(pts, g.d, i, v[u]);
      }
#pragma unroll
      for (int u = 0; u < SORT_UNR; ++u) {
        const int64_t i = base + threadIdx.x + static_cast<int64_t>(u) * 256;
        if (i < n) {
          double x[D];
#pragma unroll
          for (int k = 0; k < D; ++k) x[k] = static_cast<double>(v[u][k]);
          const double y = static_cast<double>(v[u][3]);
          ysq += y * y;
          int cell = 0;
          const int st = classify_d<D>(g, x, cell);
          if (st == PT_VALID) {
            atomicAdd(&hist[cell >> bsh], 1);
          } else {
            cell = -1;
            if (st == PT_OUTSIDE || st == PT_LEAVES) {
              const unsigned long long ecode =
                  (static_cast<unsigned long long>(row0 + i + 1) << 2) | static_cast<unsigned long long>(st);
              atomicMin(err, ecode);
            }
          }
          __stcs(cellid + i, cell);
        }
      }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < nb; j += blockDim.x) tcnt[tile * nb + j] = hist[j];
    __syncthreads();
  }
  const double s2 = block_sum<256>(ysq, sh);
  if (threadIdx.x == 0) yty_part[blockIdx.x] = s2;
}

// K2b.  Bucket totals: tiles are grouped TSCAN_G at a time (group sums), then one block sums
// the groups per bucket and scans: bbase[b] (first row of bucket b, bbase[nb] = rows
// binned) and sbase[b] (first slice of bucket b, sbase[nb] = slices).
constexpr int TSCAN_G = 64;
constexpr int SLICE_ROWS = 8192;  // K2d work unit

__global__ void k_tscan_groups(const int* __restrict__ tcnt, int64_t ntiles, int nb, int* __restrict__ gsum) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t ngroups = (ntiles + TSCAN_G - 1) / TSCAN_G;
  if (idx >= ngroups * nb) return;
  const int64_t gi = idx / nb;
  const int b = static_cast<int>(idx - gi * nb);
  const int64_t t1 = imin64((gi + 1) * TSCAN_G, ntiles);
  int s2 = 0;
  const int64_t t0 = gi * TSCAN_G;
#pragma unroll 16
  for (int q = 0; q < TSCAN_G; ++q) s2 += t0 + q < t1 ? tcnt[(t0 + q) * nb + b] : 0;
  gsum[idx] = s2;
}

// Exclusive scan of one int64 per thread over a 1024-thread block; *total = Σ.
__device__ __forceinline__ int64_t block_exscan_1024(int64_t v, int64_t* wsum, int64_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __syncthreads();
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    int64_t x = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    wsum[lane] = x;  // inclusive over warps
  }
  __syncthreads();
  *total = wsum[31];
  return incl - v + (w > 0 ? wsum[w - 1] : 0);
}

// One block (1024 threads), nb ≤ 8 · 1024.
__global__ void __launch_bounds__(1024) k_tscan_buckets(int* __restrict__ gsum, int64_t ngroups, int nb,
                                                        int64_t* __restrict__ bbase, int64_t* __restrict__ sbase) {
  __shared__ int64_t wsum[32];
  const int per = (nb + 1023) / 1024;
  const int b0 = threadIdx.x * per;
  int64_t tots[8], rows_local = 0, slices_local = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    tots[q] = 0;
    const int b = b0 + q;
    if (q < per && b < nb) {
      int64_t run = 0;
      for (int64_t gi = 0; gi < ngroups; ++gi) {  // in place: exclusive prefix over the groups
        const int v = gsum[gi * nb + b];
        gsum[gi * nb + b] = static_cast<int>(run);
        run += v;
      }
      tots[q] = run;
      rows_local += run;
      slices_local += (run + SLICE_ROWS - 1) / SLICE_ROWS;
    }
  }
  int64_t rows_total = 0, slices_total = 0;
  int64_t rrun = block_exscan_1024(rows_local, wsum, &rows_total);
  int64_t srun = block_exscan_1024(slices_local, wsum, &slices_total);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int b = b0 + q;
    if (q < per && b < nb) {
      bbase[b] = rrun;
      sbase[b] = srun;
      rrun += tots[q];
      srun += (tots[q] + SLICE_ROWS - 1) / SLICE_ROWS;
    }
  }
  if (threadIdx.x == 0) {
    bbase[nb] = rows_total;
    sbase[nb] = slices_total;
  }
}

// Tile offsets: tcnt[tile][b] ← first output row of tile's bucket-b rows = bbase[b] + rows
// of bucket b in earlier tiles (the groups' exclusive prefix from k_tscan_buckets plus the
// earlier tiles of the group) — every tile's runs are placed by row order, not by which block
// claimed a cursor first.  One warp per (group, bucket): lane l scans tiles 2l, 2l + 1 of the
// group (TSCAN_G = 64), a warp scan adds the earlier lanes (a thread walking the group's 64
// tiles serially was latency-bound: 124 µs at config 3).
static_assert(TSCAN_G == 64, "k_tile_offsets: two tiles per lane");
__global__ void k_tile_offsets(int* __restrict__ tcnt, int64_t ntiles, int nb, const int* __restrict__ gpre,
                               const int64_t* __restrict__ bbase) {
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t ngroups = (ntiles + TSCAN_G - 1) / TSCAN_G;
  if (wid >= ngroups * nb) return;
  const int64_t gi = wid / nb;
  const int b = static_cast<int>(wid - gi * nb);
  const int64_t t0 = gi * TSCAN_G + 2 * lane;
  const int v0 = t0 < ntiles ? tcnt[t0 * nb + b] : 0;
  const int v1 = t0 + 1 < ntiles ? tcnt[(t0 + 1) * nb + b] : 0;
  int incl = v0 + v1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int run = static_cast<int>(bbase[b]) + gpre[wid] + incl - v0 - v1;
  if (t0 < ntiles) tcnt[t0 * nb + b] = run;
  if (t0 + 1 < ntiles) tcnt[(t0 + 1) * nb + b] = run + v0;
}

// K2c.  The binning moves 8-byte keys (cell, row index), never the rows: K1 later gathers
// each row from the caller's layout through the sorted indices (RowSrc).  Keys are taken in
// sub-tiles of R (R = keys_per_thread · PART_NT): each sub-tile is counting-sorted by bucket
// in shared memory with deterministic ranks, placed at the tile's per-bucket offsets (row
// order, from the tile scan), and written out linearly — consecutive lanes store consecutive
// keys of a run.  (Moving the 16-byte rows twice through the two sorts cost 2.4× the bytes;
// keys stored straight from registers, every lane of a warp in a different bucket, were
// bound by the stores' address spread, not the bytes.)
template <int RPT, bool DET>
__global__ void __launch_bounds__(PART_NT, PART_MINB) k_partition(const int* __restrict__ cellid, int64_t n, int bsh,
                                                                  int nb, const int* __restrict__ toff,
                                                                  int* __restrict__ cid1, int* __restrict__ idx1,
                                                                  int kbits, BinGate gate) {
  constexpr int R = RPT * PART_NT;
  constexpr int NW = PART_NT / 32;
  static_assert(TILE_ROWS % R == 0, "a tile is a whole number of sub-tiles");
  if (gate.closed()) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  int2* stage = reinterpret_cast<int2*>(smraw);                     // (cell, row) in bucket order
  uint16_t* tab = reinterpret_cast<uint16_t*>(stage + R);           // [NW][nb] per-warp counts (det ranks)
  int* cnt = reinterpret_cast<int*>(tab + (DET ? ((nb * NW + 1) & ~1) : 0));  // per-bucket count, then local start
  int* goff = cnt + nb;    // global slot of stage key j = goff[bucket] + j
  int* gcur = goff + nb;   // next global slot of each bucket in this tile
  __shared__ int wsum[32];
  __shared__ int total_s;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (DET)
    for (int j = threadIdx.x; j < nb * NW / 2; j += PART_NT) reinterpret_cast<int*>(tab)[j] = 0;
  const int64_t ntiles = (n + TILE_ROWS - 1) / TILE_ROWS;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    for (int j = threadIdx.x; j < nb; j += PART_NT) gcur[j] = toff[tile * nb + j];
    for (int sub = 0; sub < TILE_ROWS / R; ++sub) {
      const int64_t base = tile * TILE_ROWS + static_cast<int64_t>(sub) * R;
      if (base >= n) break;
      for (int j = threadIdx.x; j < nb; j += PART_NT) cnt[j] = 0;
      __syncthreads();
      int c[RPT], rank[RPT];
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int64_t i = base + static_cast<int64_t>(u) * PART_NT + threadIdx.x;
        c[u] = i < n ? __ldcs(cellid + i) : -1;
      }
      // ranks within each bucket: deterministic (warp table) or shared-atomic cursors
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int key = c[u] >= 0 ? c[u] >> bsh : -1;
        if (DET) rank[u] = warp_rank(key, kbits, tab + w * nb);
        else rank[u] = key >= 0 ? atomicAdd(&cnt[key], 1) : 0;
      }
      __syncthreads();
      if (DET)
        for (int j = threadIdx.x; j < nb; j += PART_NT) cnt[j] = col_prefix<NW>(tab, nb, j, 0);
      __syncthreads();
      // exclusive scan of cnt over the buckets (each thread a contiguous segment)
      const int per = (nb + PART_NT - 1) / PART_NT;
      const int j0 = threadIdx.x * per;
      int local = 0;
      for (int q = 0; q < per; ++q)
        if (j0 + q < nb) local += cnt[j0 + q];
      int incl = local;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) wsum[w] = incl;
      __syncthreads();
      if (w == 0) {
        int x = lane < PART_NT / 32 ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        wsum[lane] = x;
        if (lane == 31) total_s = x;
      }
      __syncthreads();
      int run = incl - local + (w > 0 ? wsum[w - 1] : 0);
      for (int q = 0; q < per; ++q) {
        const int j = j0 + q;
        if (j < nb) {
          const int k = cnt[j];
          goff[j] = gcur[j] - run;  // the tile's next slots of bucket j, in row order
          gcur[j] += k;
          cnt[j] = run;  // local start
          run += k;
        }
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        if (c[u] >= 0) {
          const int bk = c[u] >> bsh;
          const int lp = cnt[bk] + rank[u] + (DET ? tab[w * nb + bk] : 0);
          stage[lp] = make_int2(c[u], static_cast<int>(base + static_cast<int64_t>(u) * PART_NT + threadIdx.x));
        }
      }
      __syncthreads();
      const int tot = total_s;
      for (int j = threadIdx.x; j < tot; j += PART_NT) {
        const int2 e = stage[j];
        const int64_t gp = goff[e.x >> bsh] + j;
        __stcg(cid1 + gp, e.x);
        __stcg(idx1 + gp, e.y);
      }
      if (DET)
        for (int j = threadIdx.x; j < nb * NW / 2; j += PART_NT) reinterpret_cast<int*>(tab)[j] = 0;
      __syncthreads();
    }
  }
}

// K2d.  Per-bucket counting sort by cell, in slices of SLICE_ROWS rows so the work is
// uniform whatever the bucket sizes:
//   slice_count : per slice, cell histogram (shared atomics) → scnt[slice][2^bsh]
//   slice_scan  : per bucket, per cell: exclusive over the bucket's slices (in place), then
//                 over the bucket's cells → off[c]
//   slice_scatter: per slice, shared cursors off[c] + scnt[slice][c] → sorted rows.
__device__ __forceinline__ int slice_bucket(const int64_t* __restrict__ sbase, int nb, int64_t sl) {
  int lo = 0, hi = nb;  // last b with sbase[b] <= sl
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (sbase[mid] <= sl) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(256) k_slice_count(const int* __restrict__ cid1, const int64_t* __restrict__ bbase,
                                                     const int64_t* __restrict__ sbase, int bsh, int nb,
                                                     int* __restrict__ scnt, int64_t s0, BinGate gate) {
  extern __shared__ int cnt[];
  const int64_t sl = s0 + blockIdx.x;
  if (gate.closed() || sl >= sbase[nb]) return;  // grids are sized by an upper bound
  const int b = slice_bucket(sbase, nb, sl);
  const int nbin = 1 << bsh;
  const int64_t c0 = static_cast<int64_t>(b) << bsh;
  const int64_t r0 = bbase[b] + (sl - sbase[b]) * SLICE_ROWS;
  const int64_t r1 = imin64(r0 + SLICE_ROWS, bbase[b + 1]);
  for (int j = threadIdx.x; j < nbin; j += blockDim.x) cnt[j] = 0;
  __syncthreads();
  for (int64_t i0 = r0 + threadIdx.x; i0 < r1; i0 += 256 * 8) {
    int cc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = i0 + u * 256;
      cc[u] = i < r1 ? __ldcg(cid1 + i) : -1;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (cc[u] >= 0) atomicAdd(&cnt[cc[u] - c0], 1);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < nbin; j += blockDim.x) scnt[sl * nbin + j] = cnt[j];
}

// One block per bucket (1024 threads; 2^bsh ≤ 16384 cells → ≤ 16 per thread).
__global__ void __launch_bounds__(1024) k_slice_scan(int* __restrict__ scnt, const int64_t* __restrict__ bbase,
                                                     const int64_t* __restrict__ sbase, int bsh, int nb,
                                                     int64_t cells, int64_t* __restrict__ off, int b0,
                                                     BinGate gate) {
  __shared__ int64_t wsum[32];
  const int b = b0 + blockIdx.x;
  if (gate.closed()) return;
  const int nbin = 1 << bsh;
  const int64_t c0 = static_cast<int64_t>(b) << bsh;
  const int ncell = static_cast<int>(imin64(nbin, cells - c0));
  const int64_t s0 = sbase[b], s1 = sbase[b + 1];
  const int per = (nbin + 1023) / 1024;
  const int j0 = threadIdx.x * per;
  int tot[16];
  int64_t local = 0;
  for (int q = 0; q < 16; ++q) {
    tot[q] = 0;
    const int j = j0 + q;
    if (q < per && j < ncell) {
      int run = 0;
      for (int64_t sb = s0; sb < s1; sb += 8) {  // batched: in-place stores alias the loads
        int v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = sb + u < s1 ? scnt[(sb + u) * nbin + j] : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (sb + u < s1) scnt[(sb + u) * nbin + j] = run;
          run += v[u];
        }
      }
      tot[q] = run;
      local += run;
    }
  }
  int64_t total = 0;
  int64_t run = bbase[b] + block_exscan_1024(local, wsum, &total);
  for (int q = 0; q < 16; ++q) {
    const int j = j0 + q;
    if (q < per && j < ncell) {
      off[c0 + j] = run;
      run += tot[q];
    }
  }
  // boundary entry = the next bucket's first offset (same value): a K1 pass over this bucket
  // group reads off[c + 1] of its last cell before the next group's scan has run
  if (threadIdx.x == 0) off[c0 + ncell] = bbase[b + 1];
}

// Slice scatter, direct: every thread stores its row index at its cell's shared cursor.  Used
// when a slice's runs per cell are long (≥ 32 rows on average), where the stores coalesce in
// L2 anyway and the staged kernel's extra block barriers cost more.
template <bool DET>
__global__ void __launch_bounds__(256, 3) k_slice_scatter_direct(const int* __restrict__ cid1, const int* __restrict__ idx1,
                                                                 const int64_t* __restrict__ bbase,
                                                                 const int64_t* __restrict__ sbase, int bsh, int nb,
                                                                 int64_t cells, const int* __restrict__ scnt,
                                                                 const int64_t* __restrict__ off, int* __restrict__ out,
                                                                 int64_t s0, int kbits, BinGate gate) {
  constexpr int UNR = 16;
  constexpr int NW = 256 / 32;
  extern __shared__ __align__(16) int cur[];
  const int64_t sl = s0 + blockIdx.x;
  if (gate.closed() || sl >= sbase[nb]) return;
  const int b = slice_bucket(sbase, nb, sl);
  const int nbin = 1 << bsh;
  int* tot = cur + nbin;                                    // per cell: rows of this chunk
  uint16_t* tab = reinterpret_cast<uint16_t*>(tot + nbin);  // [NW][nbin] per-warp counts (det ranks)
  const int64_t c0 = static_cast<int64_t>(b) << bsh;
  const int ncell = static_cast<int>(imin64(nbin, cells - c0));
  const int64_t r0 = bbase[b] + (sl - sbase[b]) * SLICE_ROWS;
  const int64_t r1 = imin64(r0 + SLICE_ROWS, bbase[b + 1]);
  for (int j = threadIdx.x; j < ncell; j += blockDim.x)
    cur[j] = static_cast<int>(off[c0 + j]) + scnt[sl * nbin + j];  // rows per add < 2^31
  if (DET)
    for (int j = threadIdx.x; j < nbin * NW; j += blockDim.x) tab[j] = 0;
  __syncthreads();
  const int w = threadIdx.x >> 5;
  for (int64_t base = r0; base < r1; base += 256 * UNR) {  // uniform trip count (block barriers)
    int cc[UNR], ri[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t i = base + u * 256 + threadIdx.x;
      cc[u] = -1;
      if (i < r1) {
        cc[u] = __ldcs(cid1 + i);
        ri[u] = __ldcs(idx1 + i);
      }
    }
    int rank[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int key = cc[u] >= 0 ? static_cast<int>(cc[u] - c0) : -1;
      if (DET) rank[u] = warp_rank(key, kbits, tab + w * nbin);
      else rank[u] = key >= 0 ? atomicAdd(&cur[key], 1) : 0;
    }
    if (DET) {  // per cell: each warp's slots start at cur + the earlier warps' counts
      __syncthreads();
      for (int j = threadIdx.x; j < ncell; j += blockDim.x) tot[j] = col_prefix<NW>(tab, nbin, j, 0);
      __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (cc[u] >= 0) {
        const int key = static_cast<int>(cc[u] - c0);
        const int pos = DET ? cur[key] + tab[w * nbin + key] + rank[u] : rank[u];
        out[pos] = ri[u];
      }
    }
    if (DET) {
      __syncthreads();
      for (int j = threadIdx.x; j < ncell; j += blockDim.x) cur[j] += tot[j];
      for (int j = threadIdx.x; j < nbin * NW; j += blockDim.x) tab[j] = 0;
      __syncthreads();
    }
  }
}

// Slice scatter, staged: the slice (≤ SLICE_ROWS keys) is counting-sorted by cell in shared
// memory (deterministic ranks, block scan) and written out linearly, so consecutive lanes
// store consecutive indices of one cell's run (stores straight from registers sent every lane
// of a warp to a different cell: partial-sector writes and DRAM read-modify-writes at
// config 4's ~8-row runs).
constexpr int SS_NT = 512;
constexpr int SS_RPT = SLICE_ROWS / SS_NT;

size_t slice_scatter_smem(int nbin, bool det) {
  return static_cast<size_t>(SLICE_ROWS) * (sizeof(int) + sizeof(uint16_t)) +
         2 * sizeof(int) * (static_cast<size_t>(nbin) + 1) +
         (det ? sizeof(uint16_t) * static_cast<size_t>(nbin) * (SS_NT / 32) : 0);
}

template <bool DET>
__global__ void __launch_bounds__(SS_NT, 2) k_slice_scatter(const int* __restrict__ cid1, const int* __restrict__ idx1,
                                                            const int64_t* __restrict__ bbase,
                                                            const int64_t* __restrict__ sbase, int bsh, int nb,
                                                            int64_t cells, const int* __restrict__ scnt,
                                                            const int64_t* __restrict__ off, int* __restrict__ out,
                                                            int64_t s0, int kbits, BinGate gate) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int64_t sl = s0 + blockIdx.x;
  if (gate.closed() || sl >= sbase[nb]) return;
  const int b = slice_bucket(sbase, nb, sl);
  const int nbin = 1 << bsh;
  const int64_t c0 = static_cast<int64_t>(b) << bsh;
  const int ncell = static_cast<int>(imin64(nbin, cells - c0));
  int* stage_i = reinterpret_cast<int*>(smraw);
  uint16_t* stage_c = reinterpret_cast<uint16_t*>(stage_i + SLICE_ROWS);
  int* cnt = reinterpret_cast<int*>(stage_c + SLICE_ROWS);  // per cell: count, then local start; [ncell] = total
  int* gcur = cnt + nbin + 1;                               // per cell: first global slot of this slice
  constexpr int NW = SS_NT / 32;
  uint16_t* tab = reinterpret_cast<uint16_t*>(gcur + nbin + 1);  // [NW][nbin] per-warp counts (det ranks)
  __shared__ int wsum[SS_NT / 32];
  const int64_t r0 = bbase[b] + (sl - sbase[b]) * SLICE_ROWS;
  const int nr = static_cast<int>(imin64(SLICE_ROWS, bbase[b + 1] - r0));
  for (int j = threadIdx.x; j < ncell; j += SS_NT) {
    gcur[j] = static_cast<int>(off[c0 + j]) + scnt[sl * nbin + j];  // rows per add < 2^31
    cnt[j] = 0;
  }
  if (DET)
    for (int j = threadIdx.x; j < nbin * NW; j += SS_NT) tab[j] = 0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  int ri[SS_RPT], lc[SS_RPT];  // lc: local cell, then (local cell << 16) | rank (registers: no spills)
#pragma unroll
  for (int u = 0; u < SS_RPT; ++u) {
    const int i = u * SS_NT + threadIdx.x;
    lc[u] = -1;
    if (i < nr) {
      lc[u] = static_cast<int>(__ldcs(cid1 + r0 + i) - c0);
      ri[u] = __ldcs(idx1 + r0 + i);
    }
  }
#pragma unroll
  for (int u = 0; u < SS_RPT; ++u) {  // ranks within each cell: deterministic (warp table) or atomic
    const int rank = DET ? warp_rank(lc[u], kbits, tab + w * nbin) : (lc[u] >= 0 ? atomicAdd(&cnt[lc[u]], 1) : 0);
    if (lc[u] >= 0) lc[u] = (lc[u] << 16) | rank;
  }
  __syncthreads();
  if (DET) {
    for (int j = threadIdx.x; j < ncell; j += SS_NT) cnt[j] = col_prefix<NW>(tab, nbin, j, 0);
    __syncthreads();
  }
  // exclusive scan of cnt[0..ncell) (each thread a contiguous segment)
  const int per = (ncell + SS_NT - 1) / SS_NT;
  const int j0 = threadIdx.x * per;
  int local = 0;
  for (int q = 0; q < per; ++q)
    if (j0 + q < ncell) local += cnt[j0 + q];
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    int x = lane < SS_NT / 32 ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane < SS_NT / 32) wsum[lane] = x;
  }
  __syncthreads();
  int run = incl - local + (w > 0 ? wsum[w - 1] : 0);
  for (int q = 0; q < per; ++q) {
    const int j = j0 + q;
    if (j < ncell) {
      const int k = cnt[j];
      cnt[j] = run;
      run += k;
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < SS_RPT; ++u) {
    if (lc[u] >= 0) {
      const int c = lc[u] >> 16;
      const int lp = cnt[c] + (lc[u] & 0xffff) + (DET ? tab[w * nbin + c] : 0);
      stage_i[lp] = ri[u];
      stage_c[lp] = static_cast<uint16_t>(c);
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < nr; j += SS_NT) {
    const int c = stage_c[j];
    out[static_cast<int64_t>(gcur[c]) + (j - cnt[c])] = stage_i[j];
  }
}

// Deterministic Σ of the per-block y² partials into the running yty.
__global__ void k_sum_partials(const double* __restrict__ part, int np, double* __restrict__ acc) {
  __shared__ double sh[8];
  double v = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) v += part[i];
  const double s = block_sum<256>(v, sh);
  if (threadIdx.x == 0) *acc += s;
}

// ------------------------------------------------------------------ K1 helpers
// Largest c in [lo, hi) with off[c] <= p, given off[lo] <= p < off[hi] (hi may be the end
// sentinel).  Warp-cooperative: the 32 lanes probe 32 evenly spaced offsets per round, so a
// search over 1e5+ cells costs 4 dependent loads instead of ~17 (warp-uniform call).
__device__ __forceinline__ int64_t warp_find_cell(const int64_t* __restrict__ off, int64_t lo, int64_t hi, int64_t p,
                                                  int lane) {
  while (hi - lo > 1) {
    const int64_t step = (hi - lo + 31) >> 5;
    const int64_t j = lo + step * (lane + 1);  // lane 31 probes ≥ hi
    const unsigned gt = __ballot_sync(0xffffffffu, j >= hi || off[j] > p);
    const int f = __ffs(gt) - 1;  // first probe past p; probe f − 1 (or lo) is ≤ p
    const int64_t nhi = min(hi, lo + step * (f + 1));
    lo += step * f;
    hi = nhi;
  }
  return lo;
}

// Cell of row p for a warp walking sorted rows forward from cell c (off[c] <= p): one
// coalesced probe of the next 32 offsets (consecutive cells, usually the answer), then
// the cooperative search over the rest.  A per-lane binary search per cell boundary cost
// ~20 dependent loads, which dominated sparse grids and small batches.
__device__ __forceinline__ int64_t next_cell(const int64_t* __restrict__ off, int64_t c, int64_t p, int64_t cells,
                                             int lane) {
  const int64_t j = c + 1 + lane;
  const unsigned gt = __ballot_sync(0xffffffffu, j >= cells || off[j] > p);
  if (gt) return c + __ffs(gt) - 1;
  return warp_find_cell(off, c + 32, cells, p, lane);
}

// Cell of row r0 in [c_lo, cells) (off[c_lo] <= r0 < off[cells]).
__device__ __forceinline__ int64_t first_cell(const int64_t* __restrict__ off, int64_t c_lo, int64_t cells, int64_t r0,
                                              int lane) {
  return warp_find_cell(off, c_lo, cells, r0, lane);
}

// Recompute (t_0..t_{d-1}) of a sorted (valid) row: same snap decision as classify_d, t to
// within a few ulp of the reference's (exact division in the rare snap band).
template <typename T>
__device__ __forceinline__ void row_t(const GridDev& g, const Row4<T>& r, double* t, double& y) {
#pragma unroll
  for (int k = 0; k < GSGPC_MAX_DIM; ++k) {
    if (k < g.d) {
      const double x = static_cast<double>(r.v[k]);
      double uu = __dsub_rn(x, g.mn[k]) * g.isp[k];
      const double rr = rint(uu);
      const double dd = fabs(uu - rr);
      // sorted rows are in-grid (0 ≤ u ≤ size − 1): the per-row rounding bound
      // 1e-12 + |u|·2^-48 is at most its value at u = size, a loop invariant
      const double e = 1e-12 + static_cast<double>(g.sz[k]) * 3.552713678800501e-15;
      if (dd >= 1e-9 - e && dd <= 1e-9 + e) {
        int64_t i0;
        stencil_dim(x, g.mn[k], g.sp[k], g.sz[k], i0, t[k]);
      } else {
        if (dd < 1e-9) uu = rr;
        const double i0 = fmin(floor(uu), static_cast<double>(g.sz[k] - 2));
        t[k] = uu - i0;
      }
    }
  }
  y = static_cast<double>(r.v[3]);
}

// Moment flushes are fire-and-forget reductions (RED.ADD.F64): a load-add-store of a cell
// the warp owns stalled the warp on a DRAM read per boundary, which dominated sparse cells
// (config 3, 2.56e6 rows: K1 1.65 → 0.49 ms; the 1.2e8-row step is unchanged).
__device__ __forceinline__ void flush_val(double* p, double v) { atomicAdd(p, v); }

// Bitwise-reproducible flushes.  Rows reach K1 in a fixed order (deterministic binning), each
// warp sums its fixed row range in that order, and every cell gets exactly ONE add per launch:
//   * a segment whose cell starts inside the warp's range is flushed as before (one RED per
//     entry — the only add of this launch to those addresses, so old + v is order-free);
//   * the first segment of a range whose cell started in an earlier warp's range stores its
//     partial in the warp's split record sv[warp] (scell[warp] = the cell) instead;
//   * k_split_fix then adds each split cell's chain of records, in warp order, with one add.
// (RED flushes from several warps into one cell summed in arrival order: run-to-run
// differences of ~1e-14, enough to move CG iteration counts on ill-conditioned systems.)
struct SplitRec {
  double* v;        // nwarps × rec doubles
  int64_t* cell;    // nwarps: the cell of the warp's stored partial, or −1
  __device__ __forceinline__ void none(int64_t warp, int lane) const {
    if (lane == 0) cell[warp] = -1;
  }
};

// chain heads: warps whose record continues cell c and whose predecessor's record is not c
__global__ void __launch_bounds__(128) k_split_fix(const double* __restrict__ sv, const int64_t* __restrict__ scell,
                                                   int64_t nwarps, int rec, int qv, double* __restrict__ M,
                                                   int64_t mstride, int64_t mbase, BinGate gate) {
  if (gate.closed()) return;
  const int lane = threadIdx.x & 31;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w >= nwarps) return;
  const int64_t c = scell[w];
  if (c < 0 || (w > 0 && scell[w - 1] == c)) return;
  int64_t e = w + 1;
  while (e < nwarps && scell[e] == c) ++e;
  for (int q = lane; q < qv; q += 32) {
    double s2 = 0.0;
    for (int64_t k = w; k < e; ++k) s2 += sv[k * rec + q];
    M[c * mstride + mbase + q] += s2;
  }
}

// ------------------------------------------------------------------ W^T W structure
// The reference's W^T W holds an entry for every node pair to which some point gives two
// nonzero weights (interp.cpp:188-200; zero weights are dropped, interp.cpp:94-99), however
// small the sum.  The moment reconstruction can round such a sum (e.g. the corner pair of a
// one-point cell with t ≈ 1: ~1e-17) to exactly 0, so the structure is tracked apart from
// the values: per cell, which zero-weight patterns its rows had.  Per dimension a row is
// interior (0 < t < 1: every stencil weight nonzero), on its cell's first node (t == 0:
// only slot W/2 − 1 nonzero) or on its last (t == 1, u == size − 1: only slot W/2);
// pattern p = Σ_k p_k 3^k, one byte per (cell, pattern), 0/1 — idempotent stores, merged by
// OR (MAX over ranks).  K_TOUCHED turns the patterns into the stencil's structure.
__device__ __forceinline__ int dim_pat(double t) { return t == 0.0 ? 1 : (t == 1.0 ? 2 : 0); }

template <int D>
__device__ __forceinline__ unsigned pat_bit(const double* t) {
  int p = 0;
#pragma unroll
  for (int k = D - 1; k >= 0; --k) p = p * 3 + dim_pat(t[k]);
  return 1u << p;
}

// lane p < P writes byte p of the cell's pattern record when bit p of mask is set
__device__ __forceinline__ void flush_pat(uint8_t* __restrict__ pat, int64_t c, int P, unsigned mask, int lane) {
  if (lane < P && ((mask >> lane) & 1u)) pat[c * P + lane] = 1;
}

// ------------------------------------------------------------------ K1, d = 3 cubic
// Moment record per cell: 343 x-moments + 64 y-moments; the row's powers t^0..t^6 per
// dimension are staged in shared memory (stride 26 doubles).  (Staging the y-tile operand
// products as well — stride 28 — measured slower: 5.43 vs 5.19 ms at config 3.)
constexpr int D3C_QX = 343, D3C_QY = 64, D3C_Q = 407;
static_assert(D3C_Q == D3C_QX + D3C_QY, "moment record = x-moments + y-moments");
constexpr int D3C_STRIDE = 26;

// ------------------------------------------------------------------ K1, d = 3 cubic, FP64 MMA
// The per-cell moment sums are a GEMM over the cell's points:
//   M[e0][(e1,e2)] = Σ_p t0^e0 · (t1^e1 t2^e2),   Y[a][(b,c)] = Σ_p y t0^a t1^b t2^c.
// One warp runs mma.sync.m8n8k4.f64 (D 8×8 += A 8×4 · B 4×8, k = 4 points per step):
//   x tiles t = 0..6 : A rows e0 = 0..6 plus row 7 = y  (row 7 yields Y[0][t][c]),
//                      B[k][n] = t1^t · t2^n  (n = 0..6, column 7 zero);
//   y tile (a = 1..3): A rows r < 6 → y t0^(1 + r/2) t1^(2 (r&1)),
//                      B[k][n] = t1^(n>>2) t2^(n&3)  → D[r][n] = Y[1 + r/2][2 (r&1) + (n>>2)][n&3]
//                      (48 of the 64 entries used; 8 MMAs per step for 407 moments).
// Accumulators stay in the MMA fragments (16 doubles per lane); at a cell boundary every
// lane writes its own fragment entries — no cross-lane reduction.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// The in-cell offsets of a row whose cell (digits i0[k], as doubles) is known — every row K1
// reads: t_k = (x_k − min_k)·(1/h_k) − i0_k with one rounding after the product (an FMA), to
// within 2^-52·size of the reference's (x − min)/h − i0.  Rows within 4e-9 of a cell face,
// where the reference's 1e-9 snap (interp.cpp:48-50) decides t ∈ {0, 1}, take the exact
// division.  (Re-classifying every row from scratch — rint, band test, floor, clamp — was
// ~36 FP64 instructions per row competing with the DMMAs for the FP64 pipe.)
__device__ __forceinline__ double t_exact(const GridDev& g, int k, double x) {
  int64_t i0 = 0;
  double t = 0.0;
  stencil_dim(x, g.mn[k], g.sp[k], g.sz[k], i0, t);
  return t;
}

template <typename T>
__device__ __forceinline__ void row_t_cell(const GridDev& g, const double* i0d, const Row4<T>& r, double* t,
                                           double& y) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double x = static_cast<double>(r.v[k]);
    double tk = fma(__dsub_rn(x, g.mn[k]), g.isp[k], -i0d[k]);
    if (fabs(tk - 0.5) > 0.5 - 4e-9) tk = t_exact(g, k, x);
    t[k] = tk;
  }
  y = static_cast<double>(r.v[3]);
}

template <typename T, bool PK, int MINB>
__global__ void __launch_bounds__(128, MINB) k_moments_d3c_mma(RowSrc<T, PK> pay,
                                                            const int64_t* __restrict__ off, int64_t cells,
                                                            int64_t nvalid, int64_t row0, int64_t c_lo, BinGate gate, GridDev g, double* __restrict__ mom,
                                                            uint8_t* __restrict__ pat, int64_t range, SplitRec sp) {
  __shared__ __align__(16) double sm[4][32 * D3C_STRIDE];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t warp = static_cast<int64_t>(blockIdx.x) * 4 + wib;
  if (gate.closed()) return;
  sp.none(warp, lane);
  nvalid = gate.rows(nvalid);
  const int64_t r0 = row0 + warp * range;
  if (r0 >= nvalid) return;
  const int64_t rend = min(r0 + range, nvalid);
  double* S = sm[wib];
  const int r = lane >> 2;   // A row / B column / D row
  const int kq = lane & 3;   // A column / B row: the point of the 4-point step
  const int cb = 2 * (lane & 3);  // D columns cb, cb+1
  // y-tile: A row r → (a, b_hi), B column r → (b_lo, c)
  const bool yrow = r < 6;
  const int ya = 1 + r / 2, ybh = 2 * (r & 1);
  const int ybl = r >> 2, yc = r & 3;

  double dx[7][2], dy[2];
#pragma unroll
  for (int t = 0; t < 7; ++t) dx[t][0] = dx[t][1] = 0.0;
  dy[0] = dy[1] = 0.0;
  unsigned pm = 0;  // zero-weight patterns of the cell's rows (W^T W structure)

  int64_t c = first_cell(off, c_lo, cells, r0, lane);
  int64_t p = r0;
  // rows are consumed in order; the next batch's row is loaded one batch ahead so its DRAM
  // latency hides under the current batch's MMAs (the batch after [b, b+nb) starts at b+nb)
  Row4<T> cur_row = pay[imin64(r0 + lane, rend - 1)];
  int64_t inx = pay.at(imin64(r0 + 32 + lane, rend - 1));  // the next batch's row index
  bool first = true;
  while (p < rend) {
    c = next_cell(off, c, p, cells, lane);
    const int64_t ce = off[c + 1];
    const int64_t seg_end = min(ce, rend);
    double i0d[3];  // the segment's cell digits (row-major over nc[k])
    {
      const int64_t c12 = c / g.nc[2];
      i0d[2] = static_cast<double>(c - c12 * g.nc[2]);
      const int64_t c0 = c12 / g.nc[1];
      i0d[1] = static_cast<double>(c12 - c0 * g.nc[1]);
      i0d[0] = static_cast<double>(c0);
    }
    for (int64_t b = p; b < seg_end; b += 32) {
      const int nb = static_cast<int>(imin64(32, seg_end - b));
      // the batch after [b, b + nb) starts at b + nb: its index was loaded ahead when that is
      // b + 32 (full batch); a short batch (cell end) re-reads it
      // one gather per row: only the index is re-read for a short batch (a select between two
      // gathers issued both and doubled the sectors fetched per row)
      const int64_t nix = nb == 32 ? inx : pay.at(imin64(b + nb + lane, rend - 1));
      const Row4<T> next_row = pay.row(nix);
      inx = pay.at(imin64(b + nb + 32 + lane, rend - 1));
      {
        double t[3] = {0.0, 0.0, 0.0}, y = 0.0;
        const bool v = lane < nb;
        if (v) row_t_cell<T>(g, i0d, cur_row, t, y);
        pm |= __reduce_or_sync(0xffffffffu, v ? pat_bit<3>(t) : 0u);
        double* P = S + lane * D3C_STRIDE;
        double q0 = v ? 1.0 : 0.0, q1 = q0, q2 = q0;
#pragma unroll
        for (int e = 0; e < 7; ++e) {
          P[e] = q0;
          P[8 + e] = q1;
          P[16 + e] = q2;
          q0 *= t[0];
          q1 *= t[1];
          q2 *= t[2];
        }
        P[7] = v ? y : 0.0;
      }
      __syncwarp();
      const int steps = (nb + 3) >> 2;
      for (int st = 0; st < steps; ++st) {
        const double* P = S + (4 * st + kq) * D3C_STRIDE;
        const double y = P[7];
        const double ax = P[r];            // r < 7: t0^r ; r == 7: y
        const double t2n = r < 7 ? P[16 + r] : 0.0;
        const double ay = yrow ? y * P[ya] * P[8 + ybh] : 0.0;
        const double by = P[8 + ybl] * P[16 + yc];
        const double2 p01 = *reinterpret_cast<const double2*>(P + 8);
        const double2 p23 = *reinterpret_cast<const double2*>(P + 10);
        const double2 p45 = *reinterpret_cast<const double2*>(P + 12);
        const double p6 = P[14];
        // t1^0 = 1 (0 on an empty lane, where t2n = 0 too): no multiply for tile 0
        const double bt[7] = {t2n, t2n * p01.y, t2n * p23.x, t2n * p23.y,
                              t2n * p45.x, t2n * p45.y, t2n * p6};
        (void)p01.x;
#pragma unroll
        for (int tt = 0; tt < 7; ++tt) dmma(dx[tt][0], dx[tt][1], ax, bt[tt]);
        dmma(dy[0], dy[1], ay, by);
      }
      __syncwarp();
      cur_row = next_row;
    }
    // flush this lane's fragment entries (a cell continued from the previous warp's range:
    // into the split record, see SplitRec)
    const bool split = first && off[c] < r0;
    first = false;
    double* M = split ? sp.v + warp * D3C_Q : mom + c * D3C_Q;
    auto put = [&](int q, double v) {
      if (split) M[q] = v;
      else flush_val(M + q, v);
    };
#pragma unroll
    for (int tt = 0; tt < 7; ++tt) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int col = cb + i;
        if (col < 7) {
          if (r < 7) {
            put(r * 49 + tt * 7 + col, dx[tt][i]);
          } else if (tt < 4 && col < 4) {
            put(D3C_QX + tt * 4 + col, dx[tt][i]);  // Y[a=0][b=tt][c=col]
          }
        }
        dx[tt][i] = 0.0;
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int col = cb + i;
      if (yrow) put(D3C_QX + ya * 16 + (ybh + (col >> 2)) * 4 + (col & 3), dy[i]);
      dy[i] = 0.0;
    }
    if (split && lane == 0) sp.cell[warp] = c;
    flush_pat(pat, c, 27, pm, lane);
    pm = 0;
    p = seg_end;
  }
}

// ------------------------------------------------------------------ K1, d = 2 cubic, FP64 MMA
// M[a][b] = Σ t0^a t1^b (a, b ≤ 6), Y[a][b] = Σ y t0^a t1^b (a, b ≤ 3), 2 mma.sync.m8n8k4.f64
// per 4 rows:
//   X tile: A rows a = 0..6 → t0^a, row 7 → y;  B[k][n] = t1^n (n < 7) → M and Y[0][n];
//   Y tile: A row r → (y t0) · t0^r (rows r < 3 used); same B → Y[1..3][n] (n < 4).
// Rows are staged 32 at a time regardless of cell boundaries, and each cell segment inside the
// batch runs masked steps, so sparse cells (1–100 rows, config 4) cost one step and one flush of
// the lane's fragment entries — no cross-lane reduction (the lane kernel's 65 warp sums per
// cell and 248 registers made it latency-bound).
// Cell segments come from the cells the lanes recompute for their own rows (row_tc: the same
// exact classification as K2a), compared across neighbouring lanes — no off[] lookups on the
// critical path.  Staged row R keeps element e at R·16 + (e ^ swz(R)): the staging stores (one
// row per lane) and the fragment loads (4 rows × 8 elements per step) are both conflict-free
// (2 wavefronts per 32 doubles; the odd stride-17 layout it replaces cost 3.7 per load and
// bound the kernel on the shared-memory pipe at config 4).
constexpr int D2C_QX = 49, D2C_Q = 49 + 16;

// A 64-bit shared load is served per half-warp (16 lanes = 4 elements × the step's 4 rows), so the
// rows' swizzles must differ in the 8-block bit (row bit 0) AND the 4-block bit (row bit 1);
// the low two bits take row bits 2-3, which keeps the map a bijection of the row mod 16 (the
// staging stores, one row per lane, stay conflict-free).  With ((R >> 1) & 7) in the low bits the
// rows kq = 0 and kq = 2 of a step shared a 4-block: 4 wavefronts per fragment load instead of 2
// (ncu source page: 7.4 vs 3.7 per batch and load).
__device__ __forceinline__ int d2c_swz(int R) { return ((R & 1) << 3) | (((R >> 1) & 1) << 2) | ((R >> 2) & 3); }

// row_t plus the flat cell of the row (classify's numbering: row-major over nc[k]).
template <typename T>
__device__ __forceinline__ int row_tc(const GridDev& g, const Row4<T>& r, double* t, double& y) {
  int cell = 0;
#pragma unroll
  for (int k = 0; k < GSGPC_MAX_DIM; ++k) {
    if (k < g.d) {
      const double x = static_cast<double>(r.v[k]);
      double uu = __dsub_rn(x, g.mn[k]) * g.isp[k];
      const double rr = rint(uu);
      const double dd = fabs(uu - rr);
      const double e = 1e-12 + static_cast<double>(g.sz[k]) * 3.552713678800501e-15;
      int i0;
      if (dd >= 1e-9 - e && dd <= 1e-9 + e) {
        int64_t j0;
        stencil_dim(x, g.mn[k], g.sp[k], g.sz[k], j0, t[k]);
        i0 = static_cast<int>(j0);
      } else {
        if (dd < 1e-9) uu = rr;
        const double f = fmin(floor(uu), static_cast<double>(g.sz[k] - 2));
        t[k] = uu - f;
        i0 = static_cast<int>(f);
      }
      cell = cell * static_cast<int>(g.nc[k]) + i0;
    }
  }
  y = static_cast<double>(r.v[3]);
  return cell;
}

template <typename T, bool PK>
__global__ void __launch_bounds__(128) k_moments_d2c_mma(RowSrc<T, PK> pay, int64_t nvalid,
                                                         int64_t row0, BinGate gate, GridDev g,
                                                         double* __restrict__ mom, uint8_t* __restrict__ pat,
                                                         int64_t range, SplitRec sp) {
  __shared__ __align__(16) double sm[4][32 * 16];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t warp = static_cast<int64_t>(blockIdx.x) * 4 + wib;
  if (gate.closed()) return;
  sp.none(warp, lane);
  nvalid = gate.rows(nvalid);
  const int64_t r0 = row0 + warp * range;
  if (r0 >= nvalid) return;
  const int64_t rend = min(r0 + range, nvalid);
  double* S = sm[wib];
  const int r = lane >> 2, cb = 2 * (lane & 3);
  double dx0 = 0.0, dx1 = 0.0, dy0 = 0.0, dy1 = 0.0;
  int open = -1;   // cell held in the fragments
  unsigned pm = 0;  // its rows' zero-weight patterns (W^T W structure)
  // the cell of the row before the range: a first cell equal to it continues the previous
  // warp's range (its partial goes to the split record, see SplitRec)
  int prev_cell = -1;
  if (r0 > row0) {
    double t0[3] = {0.0, 0.0, 0.0}, y0 = 0.0;
    prev_cell = row_tc<T>(g, pay[r0 - 1], t0, y0);
  }
  bool first = true;
  auto flush = [&]() {
    flush_pat(pat, open, 9, pm, lane);
    pm = 0;
    const bool split = first && open == prev_cell;
    first = false;
    double* M = split ? sp.v + warp * D2C_Q : mom + static_cast<int64_t>(open) * D2C_Q;
    auto put = [&](int q, double v) {
      if (split) M[q] = v;
      else flush_val(M + q, v);
    };
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int col = cb + i;
      const double vx = i == 0 ? dx0 : dx1, vy = i == 0 ? dy0 : dy1;
      if (col < 7 && r < 7) put(r * 7 + col, vx);
      else if (r == 7 && col < 4) put(D2C_QX + col, vx);  // Y[0][col]
      if (r < 3 && col < 4) put(D2C_QX + (r + 1) * 4 + col, vy);
    }
    if (split && lane == 0) sp.cell[warp] = open;
    dx0 = dx1 = dy0 = dy1 = 0.0;
  };
  // rows are gathered two batches ahead and their indices three batches ahead: each batch
  // waits on no load issued in it, and every lane keeps two row gathers in flight (the
  // memory-bound d = 2 K1 was latency-bound on one gather per lane: config 4 2.98 ms per
  // 1.25e8 rows with one batch of look-ahead)
  Row4<T> cur = pay[imin64(r0 + lane, rend - 1)];
  Row4<T> nxt = pay[imin64(r0 + 32 + lane, rend - 1)];
  int64_t inx = pay.at(imin64(r0 + 64 + lane, rend - 1));
  for (int64_t b = r0; b < rend; b += 32) {
    const int nb = static_cast<int>(imin64(32, rend - b));
    const Row4<T> nxt2 = pay.row(inx);
    inx = pay.at(imin64(b + 96 + lane, rend - 1));
    const bool v = lane < nb;
    int cell = 0x7fffffff;
    unsigned bit = 0;
    {
      double t[3] = {0.0, 0.0, 0.0}, y = 0.0;
      if (v) {
        cell = row_tc<T>(g, cur, t, y);
        bit = pat_bit<2>(t);
      }
      double* P = S + lane * 16;
      const int sw = d2c_swz(lane);
      double q0 = v ? 1.0 : 0.0, q1 = q0;
#pragma unroll
      for (int e = 0; e < 7; ++e) {
        P[e ^ sw] = q0;
        P[(8 + e) ^ sw] = q1;
        q0 *= t[0];
        q1 *= t[1];
      }
      P[7 ^ sw] = v ? y : 0.0;
      P[15 ^ sw] = v ? y * t[0] : 0.0;
    }
    __syncwarp();
    const int prev = __shfl_up_sync(0xffffffffu, cell, 1);
    unsigned starts = __ballot_sync(0xffffffffu, v && (lane == 0 || cell != prev));
    while (starts) {
      const int s0 = __ffs(starts) - 1;
      starts &= starts - 1;
      const int s1 = starts ? __ffs(starts) - 1 : nb;
      const int sc = __shfl_sync(0xffffffffu, cell, s0);
      if (sc != open) {
        if (open >= 0) flush();
        open = sc;
      }
      pm |= __reduce_or_sync(0xffffffffu, lane >= s0 && lane < s1 ? bit : 0u);
      const int steps = (s1 - s0 + 3) >> 2;
      for (int st = 0; st < steps; ++st) {
        const int R = s0 + 4 * st + (lane & 3);
        const int Rc = R & 31;  // masked tail rows wrap onto staged (finite) rows
        const double* P = S + Rc * 16;
        const int sw = d2c_swz(Rc);
        const double axr = P[r ^ sw];
        const double bx = P[(8 + r) ^ sw];
        const double yt = P[15 ^ sw];
        const bool ok = R < s1;
        const double ax = ok ? axr : 0.0;
        const double ay = ok ? yt * axr : 0.0;
        dmma(dx0, dx1, ax, bx);
        dmma(dy0, dy1, ay, bx);
      }
    }
    __syncwarp();
    cur = nxt;
    nxt = nxt2;
  }
  // the open cell may continue in the next warp's range: that warp records its own part
  if (open >= 0) flush();
}

// ------------------------------------------------------------------ K1, generic (lane per point)
// d ≤ 2 (any scheme) and d = 3 linear: every lane accumulates all QX + QY moments of its
// own points in registers; a segment flush warp-reduces them (butterfly) and the lanes
// write the cell's contiguous moments cooperatively.
template <int D, int W, typename T, bool PK>
__global__ void __launch_bounds__(128) k_moments_lane(RowSrc<T, PK> pay,
                                                     const int64_t* __restrict__ off, int64_t cells,
                                                     int64_t nvalid, int64_t row0, int64_t c_lo, BinGate gate, GridDev g,
                                                     double* __restrict__ mom, uint8_t* __restrict__ pat, int64_t range,
                                                     SplitRec sp) {
  constexpr int E = 2 * W - 1;
  constexpr int NP = D == 1 ? 3 : (D == 2 ? 9 : 27);
  constexpr int QX = D == 1 ? E : (D == 2 ? E * E : E * E * E);
  constexpr int QY = D == 1 ? W : (D == 2 ? W * W : W * W * W);
  constexpr int Q = QX + QY;
  const int lane = threadIdx.x & 31;
  const int64_t warp = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (gate.closed()) return;
  sp.none(warp, lane);
  nvalid = gate.rows(nvalid);
  const int64_t r0 = row0 + warp * range;
  if (r0 >= nvalid) return;
  const int64_t rend = min(r0 + range, nvalid);
  double acc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = 0.0;
  int64_t c = first_cell(off, c_lo, cells, r0, lane);
  int64_t p = r0;
  bool first = true;
  while (p < rend) {
    c = next_cell(off, c, p, cells, lane);
    const int64_t ce = off[c + 1];
    const int64_t seg_end = min(ce, rend);
    unsigned pl = 0;
    for (int64_t b = p + lane; b < seg_end; b += 32) {
      double t[3] = {0.0, 0.0, 0.0}, y = 0.0;
      row_t<T>(g, pay[b], t, y);
      pl |= pat_bit<D>(t);
      double pw[D][E];
#pragma unroll
      for (int k = 0; k < D; ++k) {
        double q = 1.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          pw[k][e] = q;
          q *= t[k];
        }
      }
      if constexpr (D == 1) {
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] += pw[0][e];
#pragma unroll
        for (int e = 0; e < W; ++e) acc[QX + e] = fma(y, pw[0][e], acc[QX + e]);
      } else if constexpr (D == 2) {
#pragma unroll
        for (int a = 0; a < E; ++a)
#pragma unroll
          for (int b2 = 0; b2 < E; ++b2) acc[a * E + b2] = fma(pw[0][a], pw[1][b2], acc[a * E + b2]);
#pragma unroll
        for (int a = 0; a < W; ++a) {
          const double ya = y * pw[0][a];
#pragma unroll
          for (int b2 = 0; b2 < W; ++b2) acc[QX + a * W + b2] = fma(ya, pw[1][b2], acc[QX + a * W + b2]);
        }
      } else {
#pragma unroll
        for (int a = 0; a < E; ++a)
#pragma unroll
          for (int b2 = 0; b2 < E; ++b2) {
            const double ab = pw[0][a] * pw[1][b2];
#pragma unroll
            for (int c2 = 0; c2 < E; ++c2) acc[(a * E + b2) * E + c2] = fma(ab, pw[2][c2], acc[(a * E + b2) * E + c2]);
          }
#pragma unroll
        for (int a = 0; a < W; ++a)
#pragma unroll
          for (int b2 = 0; b2 < W; ++b2) {
            const double yab = y * pw[0][a] * pw[1][b2];
#pragma unroll
            for (int c2 = 0; c2 < W; ++c2)
              acc[QX + (a * W + b2) * W + c2] = fma(yab, pw[2][c2], acc[QX + (a * W + b2) * W + c2]);
          }
      }
    }
    // butterfly reduce, then lane l writes moments l, l+32, ...
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] = warp_sum(acc[q]);
    const bool split = first && off[c] < r0;
    first = false;
    double* M = split ? sp.v + warp * Q : mom + c * Q;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      if ((q & 31) == lane) {
        if (split) M[q] = acc[q];
        else flush_val(M + q, acc[q]);
      }
      acc[q] = 0.0;
    }
    if (split && lane == 0) sp.cell[warp] = c;
    flush_pat(pat, c, NP, __reduce_or_sync(0xffffffffu, pl), lane);
    p = seg_end;
  }
}

// ------------------------------------------------------------------ probe images (K1p)
// W^T v_p for P Rademacher probes: per cell, Σ_p s_p Π_k t_pk^{e_k} (e_k ≤ W-1) — the same
// y-moment reconstruction then yields W^T v_p.  Lane j owns probe j (P ≤ 64 → two passes).
template <int D, int W, typename T, bool PK>
__global__ void __launch_bounds__(64) k_probe_moments(RowSrc<T, PK> pay,
                                                      const uint64_t* __restrict__ pw,
                                                      const int64_t* __restrict__ off, int64_t cells,
                                                      int64_t nvalid, int64_t row0, int64_t c_lo, BinGate gate, GridDev g, int probes,
                                                      double* __restrict__ pmom /*cells × P × QY*/,
                                                      int64_t range, int pbase, SplitRec sp) {
  constexpr int QY = D == 1 ? W : (D == 2 ? W * W : W * W * W);
  __shared__ __align__(16) double sm[2][32 * (QY + 1)];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t warp = static_cast<int64_t>(blockIdx.x) * 2 + wib;
  if (gate.closed()) return;
  sp.none(warp, lane);
  nvalid = gate.rows(nvalid);
  const int64_t r0 = row0 + warp * range;
  if (r0 >= nvalid) return;
  const int64_t rend = min(r0 + range, nvalid);
  const int nw = (probes + 63) >> 6;
  const int pj = pbase + lane;  // probe owned by this lane
  const bool plive = pj < probes;
  double* S = sm[wib];
  uint64_t* SW = reinterpret_cast<uint64_t*>(S + 32 * QY);
  double acc[QY];
#pragma unroll
  for (int q = 0; q < QY; ++q) acc[q] = 0.0;
  int64_t c = first_cell(off, c_lo, cells, r0, lane);
  int64_t p = r0;
  bool first = true;
  while (p < rend) {
    c = next_cell(off, c, p, cells, lane);
    const int64_t ce = off[c + 1];
    const int64_t seg_end = min(ce, rend);
    for (int64_t b = p; b < seg_end; b += 32) {
      const int nb = static_cast<int>(imin64(32, seg_end - b));
      {
        double t[3] = {0.0, 0.0, 0.0}, y = 0.0;
        const bool v = lane < nb;
        if (v) row_t<T>(g, pay[b + lane], t, y);
        double pw1[D][W];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          double q = v ? 1.0 : 0.0;
#pragma unroll
          for (int e = 0; e < W; ++e) {
            pw1[k][e] = q;
            q *= t[k];
          }
        }
        double* P = S + lane * QY;
#pragma unroll
        for (int q = 0; q < QY; ++q) {
          double m = 1.0;
          int qq = q;
#pragma unroll
          for (int k = D - 1; k >= 0; --k) {
            m *= pw1[k][qq % W];
            qq /= W;
          }
          P[q] = m;
        }
        SW[lane] = v ? pw[pay.at(b + lane) * nw + (pj >> 6)] : 0ull;
      }
      __syncwarp();
      for (int r = 0; r < nb; ++r) {
        const double* P = S + r * QY;
        const uint64_t bits = SW[r];
        const double sgn = ((bits >> (pj & 63)) & 1ull) ? 1.0 : -1.0;
#pragma unroll
        for (int q = 0; q < QY; ++q) acc[q] = fma(sgn, P[q], acc[q]);
      }
      __syncwarp();
    }
    const bool split = first && off[c] < r0;
    first = false;
    if (plive) {  // split record: 32 probes × QY per warp
      double* M = split ? sp.v + (warp * 32 + lane) * QY : pmom + (c * probes + pj) * QY;
#pragma unroll
      for (int q = 0; q < QY; ++q) {
        if (split) M[q] = acc[q];
        else flush_val(M + q, acc[q]);
      }
    }
    if (split && lane == 0) sp.cell[warp] = c;
#pragma unroll
    for (int q = 0; q < QY; ++q) acc[q] = 0.0;
    p = seg_end;
  }
}

// ------------------------------------------------------------------ finalize kernels
// One separable transform along dimension k maps (cell c_k, exponent e_k) to (node a_k,
// offset δ_k) (x-moments → W^T W stencil) or to node a_k alone (y-/probe-moments → W^T y /
// W^T v_p).  A thread owns one (line, node): it loads the W·E moments of the W cells whose
// 4^d block contains the node once and produces every output offset from them.
struct XformDims {
  int sp_in, sp_out;   // Π spatial extents of input / output (< 2^31)
  int inner_sp;        // Π spatial extents of dims after k (already transformed, same in/out)
  int ext_in_k, ext_out_k;  // cells / nodes along k
  int inner_q;         // Π index extents of digits after k (same in/out)
  int shift;           // cell of node a at slot i: c = a + shift - i (cubic 1, linear 0)
  // input addressing: moment-major In[q * sp_in + sp] or cell-major In[sp * cstride + qoff + q]
  int cell_major;
  int64_t cstride, qoff;
  // output: moment-major Out[q * sp_out + sp], or the half stencil (last x pass): q >= c0 only
  int half;
  int64_t c0;
};

// Thread = (output spatial index sp: blockIdx.x/threadIdx.x, remaining index digits:
// blockIdx.y).  W (4 cubic / 2 linear) and the y/x mode are template parameters so the
// 4 × 7 load window and the coefficient loops unroll without guards; all index math is
// 32-bit (the launch is issue-bound otherwise).
template <int W, bool YM>
__global__ void __launch_bounds__(256) k_xform(const double* __restrict__ in, double* __restrict__ out, XformDims x) {
  constexpr int E = 2 * W - 1;
  constexpr int EIN = YM ? W : E;
  const int sp = blockIdx.x * blockDim.x + threadIdx.x;
  if (sp >= x.sp_out) return;
  const int qrest = blockIdx.y;
  const int q_hi = qrest / x.inner_q, q_lo = qrest - q_hi * x.inner_q;
  const int t = sp / x.inner_sp;
  const int sp_lo = sp - t * x.inner_sp;
  const int sp_hi = t / x.ext_out_k;
  const int a = t - sp_hi * x.ext_out_k;
  double v[W][EIN];
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const int c = a + x.shift - i;
    const bool ok = c >= 0 && c < x.ext_in_k;
    const int spi = (sp_hi * x.ext_in_k + c) * x.inner_sp + sp_lo;
#pragma unroll
    for (int e = 0; e < EIN; ++e) {
      const int qi = (q_hi * EIN + e) * x.inner_q + q_lo;
      const int64_t addr = x.cell_major ? static_cast<int64_t>(spi) * x.cstride + x.qoff + qi
                                        : static_cast<int64_t>(qi) * x.sp_in + spi;
      v[i][e] = ok ? __ldg(in + addr) : 0.0;
    }
  }
  if constexpr (YM) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < W; ++i)
#pragma unroll
      for (int e = 0; e < EIN; ++e) acc = fma(v[i][e], c_poly[W == 4].P[i * 4 + e], acc);
    const int qo = q_hi * x.inner_q + q_lo;  // digit k collapsed to extent 1
    out[static_cast<int64_t>(qo) * x.sp_out + sp] = acc;
  } else {
#pragma unroll
    for (int dq = 0; dq < E; ++dq) {
      const int delta = dq - (W - 1);
      const int64_t qo = static_cast<int64_t>(q_hi * E + dq) * x.inner_q + q_lo;
      if (x.half && qo < x.c0) continue;
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < W; ++i) {
        const int j = i + delta;
        if (j >= 0 && j < W) {
#pragma unroll
          for (int e = 0; e < EIN; ++e) acc = fma(v[i][e], c_poly[W == 4].C[(i * 4 + j) * 7 + e], acc);
        }
      }
      out[(x.half ? qo - x.c0 : qo) * x.sp_out + sp] = acc;
    }
  }
}

// First transform (innermost dimension k = d−1) of both chains straight from the
// cell-major moments.  Cells along the last dimension are consecutive records, so a block
// stages the records of one tile of a grid line ([cell][Q] fp64, contiguous) in shared
// memory with coalesced loads and produces every x output (node a, exponent digits before
// k, offset δ) and y output (node a, digits before k) of the tile from it — the per-thread
// k_xform read of 4 × 7 values at a 407-double stride between lanes was L1-wavefront bound.
struct XformFirst {
  int Q, QX;                 // record stride, x-moments per record (y-moments follow)
  int ext_in, ext_out;       // cells / nodes along k
  int lines;                 // Π cells of the other dimensions
  int tiles, TA;             // node tiles per line, nodes per tile
  int qx_rest, qy_rest;      // E^{d−1}, W^{d−1}
  int sp_out;                // lines × ext_out
  int shift;                 // cubic 1, linear 0
};

template <int W>
__global__ void __launch_bounds__(256, 2) k_xform_first(const double* __restrict__ mom, double* __restrict__ outx,
                                                     double* __restrict__ outy, XformFirst x) {
  constexpr int E = 2 * W - 1;
  extern __shared__ __align__(16) double stage[];
  const int line = blockIdx.x / x.tiles, tile = blockIdx.x - line * x.tiles;
  const int a0 = tile * x.TA;
  const int na = min(x.TA, x.ext_out - a0);
  const int c_lo = max(0, a0 + x.shift - (W - 1));
  const int c_hi = min(x.ext_in - 1, a0 + na - 1 + x.shift);
  // the tile's records in one bulk copy (TMA engine, no registers or warps tied up):
  // start rounded down to 16 bytes, size up to 16 bytes (the moment buffer has 2 spare doubles)
  __shared__ __align__(8) uint64_t bar;
  const int64_t first = (static_cast<int64_t>(line) * x.ext_in + c_lo) * x.Q;
  const int pre = static_cast<int>(first & 1);
  const int cnt = (c_hi - c_lo + 1) * x.Q;
  const unsigned bytes = static_cast<unsigned>(((pre + cnt + 1) & ~1) * sizeof(double));
  const unsigned bar_s = static_cast<unsigned>(__cvta_generic_to_shared(&bar));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(stage))),
                 "l"(mom + (first - pre)), "r"(bytes), "r"(bar_s)
                 : "memory");
  }
  asm volatile(
      "{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W%=;\n}\n" ::"r"(bar_s)
      : "memory");
  const double* rec = stage + pre;
  const int sp0 = line * x.ext_out + a0;
  const int nx = na * x.qx_rest;
  for (int it = threadIdx.x; it < nx; it += blockDim.x) {
    const int q_hi = it / na, ai = it - q_hi * na;
    const int a = a0 + ai;
    // per cell slot i: 7 exponents in registers, added into every offset that pairs with i
    // (same summation order as k_xform: i ascending, then e)
    double acc[E];
#pragma unroll
    for (int dq = 0; dq < E; ++dq) acc[dq] = 0.0;
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const int c = a + x.shift - i;
      if (c >= 0 && c < x.ext_in) {
        const double* r = rec + (c - c_lo) * x.Q + q_hi * E;
        double v[E];
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = r[e];
#pragma unroll
        for (int dq = 0; dq < E; ++dq) {
          const int j = i + dq - (W - 1);
          if (j >= 0 && j < W) {
#pragma unroll
            for (int e = 0; e < E; ++e) acc[dq] = fma(v[e], c_poly[W == 4].C[(i * 4 + j) * 7 + e], acc[dq]);
          }
        }
      }
    }
#pragma unroll
    for (int dq = 0; dq < E; ++dq) outx[static_cast<int64_t>(q_hi * E + dq) * x.sp_out + sp0 + ai] = acc[dq];
  }
  const int ny = na * x.qy_rest;
  for (int it = threadIdx.x; it < ny; it += blockDim.x) {
    const int q_hi = it / na, ai = it - q_hi * na;
    const int a = a0 + ai;
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const int c = a + x.shift - i;
      if (c >= 0 && c < x.ext_in) {
        const double* r = rec + (c - c_lo) * x.Q + x.QX + q_hi * W;
#pragma unroll
        for (int e = 0; e < W; ++e) acc = fma(r[e], c_poly[W == 4].P[i * 4 + e], acc);
      }
    }
    outy[static_cast<int64_t>(q_hi) * x.sp_out + sp0 + ai] = acc;
  }
}

// ================================================================== host side
// (x0[, x1[, x2]], y) rows packed 4 elements wide and vector-aligned → one vector load per row
static bool packed4(const PointsDev& p, int d, size_t es) {
  if (p.xs != 4 || p.ys != 4) return false;
  for (int k = 0; k < d; ++k)
    if (p.xo[k] != k) return false;
  const char* x = static_cast<const char*>(p.x);
  const char* y = static_cast<const char*>(p.y);
  return d == 3 && y == x + 3 * es && (reinterpret_cast<uintptr_t>(x) % (4 * es)) == 0;
}

BinDesc bin_desc(int64_t cells) {
  BinDesc bd{};
  static const int64_t target = [] {  // GSGPC_BIN_BUCKETS: diagnostics override
    const char* e = getenv("GSGPC_BIN_BUCKETS");
    return e ? std::max<int64_t>(1, atoll(e)) : int64_t{512};  // B200, config 3 partition + slice sort: 1024 2.89, 512 2.57, 256 2.58, 128 2.66 ms
  }();
  // ≥ cells / 1024 buckets: the staged slice scatter's per-warp rank tables stay ≤ 32 KB
  // (config 4, 1024² nodes: 2048-cell buckets cost 3.6 vs 1024-cell ~2.7 ms per 1.25e8 rows)
  const int64_t tgt = std::min<int64_t>(BIN_MAX_NB, std::max<int64_t>(target, (cells + 1023) / 1024));
  bd.bsh = 0;
  while (((cells + (int64_t{1} << bd.bsh) - 1) >> bd.bsh) > tgt && bd.bsh < BIN_MAX_BSH) ++bd.bsh;
  bd.nb = static_cast<int>((cells + (int64_t{1} << bd.bsh) - 1) >> bd.bsh);
  if (bd.nb > BIN_MAX_NB)  // k_tscan_buckets: ≤ 8 buckets per thread of one 1024-thread block
    throw Error(GSGPC_UNSUPPORTED, "sufficient_stats: grids above 2^14 · 8192 cells are not supported by this build");
  return bd;
}

int64_t bin_tiles(int64_t n) { return ceil_div(n, TILE_ROWS); }
int64_t bin_groups(int64_t n) { return ceil_div(bin_tiles(n), TSCAN_G); }

template <typename T, int D>
static void launch_classify_d(const Launch& L, const PointsDev& p, int64_t n, int64_t row0, const GridDev& g,
                              const BinDesc& bd, int* tcnt, unsigned long long* err, double* part, int nblk,
                              int* cellid) {
  const size_t sm = sizeof(int) * bd.nb;
  if (packed4(p, g.d, sizeof(T))) {
    k_classify_tiles<T, true, D><<<nblk, 256, sm, L.s>>>(p, n, row0, g, bd.bsh, bd.nb, tcnt, err, part, cellid);
  } else {
    k_classify_tiles<T, false, D><<<nblk, 256, sm, L.s>>>(p, n, row0, g, bd.bsh, bd.nb, tcnt, err, part, cellid);
  }
}

template <typename T>
static void launch_classify(const Launch& L, const PointsDev& p, int64_t n, int64_t row0, const GridDev& g,
                            const BinDesc& bd, int* tcnt, unsigned long long* err, double* part, int nblk,
                            int* cellid) {
  if (g.d == 1) launch_classify_d<T, 1>(L, p, n, row0, g, bd, tcnt, err, part, nblk, cellid);
  else if (g.d == 2) launch_classify_d<T, 2>(L, p, n, row0, g, bd, tcnt, err, part, nblk, cellid);
  else launch_classify_d<T, 3>(L, p, n, row0, g, bd, tcnt, err, part, nblk, cellid);
}

void run_classify(const Launch& L, int dtype, const PointsDev& p, int64_t n, int64_t row0, const GridDev& g,
                  const BinDesc& bd, int* tcnt, unsigned long long* err, double* part, int nblk, int* cellid) {
  if (dtype == GSGPC_F32) launch_classify<float>(L, p, n, row0, g, bd, tcnt, err, part, nblk, cellid);
  else launch_classify<double>(L, p, n, row0, g, bd, tcnt, err, part, nblk, cellid);
  L.count();
  GSGPC_CUDA(cudaGetLastError());
}

__global__ void k_commit_add(const unsigned long long* err, const double* src, double* dst) {
  if (*err == ~0ull) *dst += *src;
}

void run_commit_add(const Launch& L, const unsigned long long* err, const double* src, double* dst) {
  k_commit_add<<<1, 1, 0, L.s>>>(err, src, dst);
  L.count();
  GSGPC_CUDA(cudaGetLastError());
}

void run_sum_partials(const Launch& L, const double* part, int np, double* acc) {
  k_sum_partials<<<1, 256, 0, L.s>>>(part, np, acc);
  L.count();
  GSGPC_CUDA(cudaGetLastError());
}

void run_bucket_totals(const Launch& L, const BinDesc& bd, int64_t n, int* tcnt, int* gsum, int64_t* bbase,
                       int64_t* sbase) {
  const int64_t nt = bin_tiles(n), ng = bin_groups(n);
  const unsigned gb = static_cast<unsigned>(ceil_div(ng * bd.nb, 256));
  k_tscan_groups<<<gb, 256, 0, L.s>>>(tcnt, nt, bd.nb, gsum);
  k_tscan_buckets<<<1, 1024, 0, L.s>>>(gsum, ng, bd.nb, bbase, sbase);
  k_tile_offsets<<<static_cast<unsigned>(ceil_div(ng * bd.nb * 32, 256)), 256, 0, L.s>>>(tcnt, nt, bd.nb, gsum,
                                                                                       bbase);  // tcnt → per-tile offsets
  L.count(3);
  GSGPC_CUDA(cudaGetLastError());
}

int64_t bin_slices_max(int64_t nvalid, const BinDesc& bd) { return ceil_div(nvalid, SLICE_ROWS) + bd.nb; }

// Deterministic ranks while the per-warp count table fits next to the staged sub-tile (bucket
// count nb ≤ 1280: every grid up to ~2e7 cells); beyond that the shared-atomic cursors.
constexpr int DET_MAX_NB = 1280;

// Deterministic ranks: lanes sharing a key from ballots (one per key bit) or from MATCH.ANY
// (GSGPC_RANK_MATCH = "part", "slice", "both" or "none" selects MATCH.ANY per pass).
static int rank_bits(bool partition, int keybits) {
  static const int mode = [] {
    const char* e = getenv("GSGPC_RANK_MATCH");
    if (!e) return 1;  // default: MATCH.ANY in the partition, ballots in the slice scatter
    const std::string v(e);
    return v == "part" ? 1 : v == "slice" ? 2 : v == "both" ? 3 : 0;
  }();
  return (mode & (partition ? 1 : 2)) ? -1 : keybits;
}

static bool bin_nondet() {  // GSGPC_BIN_NONDET=1: diagnostics only (shared-atomic ranks, not reproducible)
  static const bool v = getenv("GSGPC_BIN_NONDET") != nullptr;
  return v;
}

template <int RPT>
static size_t partition_smem(const BinDesc& bd, bool det) {
  return static_cast<size_t>(RPT) * PART_NT * sizeof(int2) + 3 * sizeof(int) * bd.nb +
         (det ? sizeof(uint16_t) * ((static_cast<size_t>(bd.nb) * (PART_NT / 32) + 1) & ~size_t{1}) : 0);
}

template <int RPT, bool DET>
static void launch_partition_r(const Launch& L, int64_t n, const BinDesc& bd, const int* cellid, const int* toff,
                               int* cid1, int* idx1, int nblk, BinGate gate) {
  const size_t sm = partition_smem<RPT>(bd, DET);
  set_max_dynamic_smem(reinterpret_cast<const void*>(k_partition<RPT, DET>), static_cast<int>(sm));
  const int kbits = rank_bits(true, 32 - __builtin_clz(static_cast<unsigned>(std::max(bd.nb - 1, 1))));
  k_partition<RPT, DET><<<nblk, PART_NT, sm, L.s>>>(cellid, n, bd.bsh, bd.nb, toff, cid1, idx1, kbits, gate);
}

// keys per thread so that the staged sub-tile + per-bucket counters (+ rank tables) fit the
// shared memory
template <bool DET>
static void launch_partition_d(const Launch& L, int64_t n, const BinDesc& bd, const int* cellid, const int* toff,
                               int* cid1, int* idx1, int nblk, BinGate gate) {
  const size_t budget = 220 * 1024 / PART_MINB;
  if (partition_smem<32>(bd, DET) <= budget)
    launch_partition_r<32, DET>(L, n, bd, cellid, toff, cid1, idx1, nblk, gate);
  else if (partition_smem<16>(bd, DET) <= budget)
    launch_partition_r<16, DET>(L, n, bd, cellid, toff, cid1, idx1, nblk, gate);
  else if (partition_smem<8>(bd, DET) <= budget)
    launch_partition_r<8, DET>(L, n, bd, cellid, toff, cid1, idx1, nblk, gate);
  else if (partition_smem<4>(bd, DET) <= budget)
    launch_partition_r<4, DET>(L, n, bd, cellid, toff, cid1, idx1, nblk, gate);
  else
    launch_partition_r<1, DET>(L, n, bd, cellid, toff, cid1, idx1, nblk, gate);
}

void run_partition(const Launch& L, int64_t n, const BinDesc& bd, const int* cellid, const int* toff, int* cid1,
                   int* idx1, const unsigned long long* err) {
  const BinGate gate{err, nullptr};
  int dev = 0, sms = 148;
  GSGPC_CUDA(cudaGetDevice(&dev));
  GSGPC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int nblk = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(bin_tiles(n), sms * PART_MINB)));
  if (bd.nb <= DET_MAX_NB && !bin_nondet()) launch_partition_d<true>(L, n, bd, cellid, toff, cid1, idx1, nblk, gate);
  else launch_partition_d<false>(L, n, bd, cellid, toff, cid1, idx1, nblk, gate);
  L.count();
  GSGPC_CUDA(cudaGetLastError());
}

void run_slice_sort(const Launch& L, const BinDesc& bd, int64_t cells, int b0, int b1, int64_t s0, int64_t s1,
                    const int* cid1, const int* idx1, const int64_t* bbase, const int64_t* sbase, int* scnt,
                    int64_t* off, int* idx_s, const unsigned long long* err) {
  const BinGate gate{err, nullptr};
  const size_t sm = sizeof(int) * (size_t{1} << bd.bsh);
  const int64_t ns = s1 - s0;
  if (ns > 0) {
    set_max_dynamic_smem(reinterpret_cast<const void*>(k_slice_count), static_cast<int>(sm));  // 2^bsh ≤ 16384 cells
    k_slice_count<<<static_cast<unsigned>(ns), 256, sm, L.s>>>(cid1, bbase, sbase, bd.bsh, bd.nb, scnt, s0, gate);
    L.count();
  }
  if (b1 > b0)
  {
    k_slice_scan<<<static_cast<unsigned>(b1 - b0), 1024, 0, L.s>>>(scnt, bbase, sbase, bd.bsh, bd.nb, cells, off, b0, gate);
    L.count();
  }
  if (ns > 0) {
    const int nbin = 1 << bd.bsh;
    static const bool direct = [] {  // GSGPC_SLICE_DIRECT=1: diagnostics (direct scatter for long runs)
      const char* e = getenv("GSGPC_SLICE_DIRECT");
      return e && e[0] == '1';
    }();
    if (direct && SLICE_ROWS / nbin >= 32) {
      // deterministic ranks: cursors + a u16 table of 8 warps per cell (nbin ≤ 256 here)
      const size_t smd = 2 * sizeof(int) * static_cast<size_t>(nbin) + sizeof(uint16_t) * static_cast<size_t>(nbin) * 8;
      auto k = bin_nondet() ? k_slice_scatter_direct<false> : k_slice_scatter_direct<true>;
      k<<<static_cast<unsigned>(ns), 256, smd, L.s>>>(cid1, idx1, bbase, sbase, bd.bsh, bd.nb, cells, scnt, off, idx_s,
                                                       s0, rank_bits(false, bd.bsh), gate);
    } else {
      // deterministic ranks while the per-warp table (16 warps × cells, u16) fits: 2^bsh ≤ 2048
      const bool det = nbin <= 2048 && !bin_nondet();
      const size_t ssm = slice_scatter_smem(nbin, det);
      auto k = det ? k_slice_scatter<true> : k_slice_scatter<false>;
      set_max_dynamic_smem(reinterpret_cast<const void*>(k), static_cast<int>(ssm));
      k<<<static_cast<unsigned>(ns), SS_NT, ssm, L.s>>>(cid1, idx1, bbase, sbase, bd.bsh, bd.nb, cells, scnt, off,
                                                         idx_s, s0, rank_bits(false, bd.bsh), gate);
    }
  }
  L.count(ns > 0 ? 1 : 0);
  GSGPC_CUDA(cudaGetLastError());
}

int moments_per_cell(int d, int W) {
  const int E = 2 * W - 1;
  int qx = 1, qy = 1;
  for (int k = 0; k < d; ++k) {
    qx *= E;
    qy *= W;
  }
  return qx + qy;
}

// Rows per warp of the d = 3 cubic K1: large ranges mean fewer split records (one per range
// that starts inside a cell) and fewer flushes, small ones a shorter tail.  Ranges double from
// 512 up to 2048 while a launch still has ≥ 8 waves of 20 warps per SM (B200, config 3, K1 +
// split fix-up: 512 → 5.52, 1024 → 5.35, 1536 → 5.29, 2048 → 5.28, 3072 → 5.27 ms; with rows
// moved by the binning, round 1: 512 5.40, 1024 5.51 ms).  GSGPC_K1_RANGE: diagnostics.
static int64_t k1_range_d3(int64_t rows) {
  static const int64_t forced = [] {
    const char* e = getenv("GSGPC_K1_RANGE");
    return e ? std::max<int64_t>(32, atoll(e)) : int64_t{0};
  }();
  if (forced) return forced;
  const int64_t target = rows / (static_cast<int64_t>(sm_count()) * 20 * 8);
  int64_t range = 512;
  while (range * 2 <= std::min<int64_t>(2048, target)) range *= 2;
  return range;
}

// Split records (SplitRec) of one K1 / K1p launch: warps ≤ rows / min range + a block's slack.
int64_t split_rec_warps(int64_t rows) { return ceil_div(rows, std::min<int64_t>(512, k1_range_d3(rows))) + 8; }
int64_t split_rec_doubles(const GridDev& g, int probes) {
  int64_t q = moments_per_cell(g.d, g.W);
  int QY = 1;
  for (int k = 0; k < g.d; ++k) QY *= g.W;
  if (probes > 0) q = std::max<int64_t>(q, int64_t{32} * QY);
  return q;
}

static void split_fix(const Launch& L, const SplitBuf& sb, int64_t nwarps, int rec, int qv, double* M,
                      int64_t mstride, int64_t mbase, BinGate gate, SplitFixJob* defer = nullptr) {
  if (defer) {  // the caller runs it (run_split_fix), e.g. to time it apart from K1
    *defer = SplitFixJob{nwarps, rec, qv, M, mstride, mbase, gate.err, gate.rows_end, true};
    return;
  }
  if (nwarps <= 0) return;
  if (nwarps > sb.warps || rec > sb.rec) throw Error(GSGPC_RUNTIME_ERROR, "K1 split records undersized");
  k_split_fix<<<static_cast<unsigned>(ceil_div(nwarps, 4)), 128, 0, L.s>>>(sb.v, sb.cell, nwarps, rec, qv, M, mstride,
                                                                           mbase, gate);
  L.count();
}

template <typename T, bool PK>
static void launch_moments(const Launch& L, const RowSrc<T, PK>& P, const int64_t* off, int64_t row0, int64_t nvalid,
                           int64_t c_lo, int64_t c_hi, const GridDev& g, double* mom, uint8_t* pat, BinGate gate,
                           const SplitBuf& sb, SplitFixJob* defer) {
  if (nvalid <= row0) return;
  const SplitRec sp{sb.v, sb.cell};
  const int Q = moments_per_cell(g.d, g.W);
  if (g.d == 3 && g.W == 4) {
    const int64_t range = k1_range_d3(nvalid - row0);
    const int64_t warps = ceil_div(nvalid - row0, range);
    static const int minb = [] {
      const char* e = getenv("GSGPC_K1_MINB");
      return e ? atoi(e) : 5;  // resident blocks/SM (B200, config 3, row prefetch): 4, 5 → 5.36, 6 → 5.39 ms
    }();
    const unsigned blocks = static_cast<unsigned>(ceil_div(warps, 4));
    if (static_cast<int64_t>(blocks) * 4 > sb.warps) throw Error(GSGPC_RUNTIME_ERROR, "K1 split records undersized");
#define GSGPC_D3(MB) k_moments_d3c_mma<T, PK, MB><<<blocks, 128, 0, L.s>>>(P, off, c_hi, nvalid, row0, c_lo, gate, g, mom, pat, range, sp)
    if (minb >= 6) GSGPC_D3(6);
    else if (minb == 5) GSGPC_D3(5);
    else GSGPC_D3(4);
#undef GSGPC_D3
    split_fix(L, sb, static_cast<int64_t>(blocks) * 4, Q, Q, mom, Q, 0, gate, defer);
  } else if (g.d == 2 && g.W == 4) {
    const int64_t range = k1_range_d3(nvalid - row0);  // same trade-off as d = 3
    const unsigned blocks = static_cast<unsigned>(ceil_div(ceil_div(nvalid - row0, range), 4));
    if (static_cast<int64_t>(blocks) * 4 > sb.warps) throw Error(GSGPC_RUNTIME_ERROR, "K1 split records undersized");
    k_moments_d2c_mma<T, PK><<<blocks, 128, 0, L.s>>>(P, nvalid, row0, gate, g, mom, pat, range, sp);
    split_fix(L, sb, static_cast<int64_t>(blocks) * 4, Q, Q, mom, Q, 0, gate, defer);
  } else {
    const int64_t range = 1024;
    const int64_t warps = ceil_div(nvalid - row0, range);
    const unsigned blocks = static_cast<unsigned>(ceil_div(warps, 4));
    if (static_cast<int64_t>(blocks) * 4 > sb.warps) throw Error(GSGPC_RUNTIME_ERROR, "K1 split records undersized");
#define GSGPC_LM(DD, WW)                                                                          \
  if (g.d == DD && g.W == WW) {                                                                 \
    k_moments_lane<DD, WW, T, PK><<<blocks, 128, 0, L.s>>>(P, off, c_hi, nvalid, row0, c_lo, gate, g, mom, pat, range, sp); \
  }
    GSGPC_LM(1, 2) GSGPC_LM(1, 4) GSGPC_LM(2, 2) GSGPC_LM(2, 4) GSGPC_LM(3, 2)
#undef GSGPC_LM
    split_fix(L, sb, static_cast<int64_t>(blocks) * 4, Q, Q, mom, Q, 0, gate, defer);
  }
}

template <typename T>
static void launch_moments_t(const Launch& L, const PointsDev& p, const int* idx, const int64_t* off, int64_t row0,
                             int64_t nvalid, int64_t c_lo, int64_t c_hi, const GridDev& g, double* mom, uint8_t* pat,
                             BinGate gate, const SplitBuf& sb, SplitFixJob* defer) {
  if (packed4(p, g.d, sizeof(T)))
    launch_moments<T, true>(L, RowSrc<T, true>{p, idx, g.d}, off, row0, nvalid, c_lo, c_hi, g, mom, pat, gate, sb,
                            defer);
  else
    launch_moments<T, false>(L, RowSrc<T, false>{p, idx, g.d}, off, row0, nvalid, c_lo, c_hi, g, mom, pat, gate, sb,
                             defer);
}

void run_split_fix(const Launch& L, const SplitBuf& sb, const SplitFixJob& j) {
  if (!j.pending) return;
  split_fix(L, sb, j.nwarps, j.rec, j.qv, j.M, j.mstride, j.mbase, BinGate{j.err, j.rows_end});
  GSGPC_CUDA(cudaGetLastError());
}

void run_moments(const Launch& L, int dtype, const PointsDev& p, const int* idx, const int64_t* off, int64_t row0,
                 int64_t nvalid, int64_t c_lo, int64_t c_hi, const GridDev& g, double* mom, uint8_t* pat,
                 const unsigned long long* err, const SplitBuf& sb, const int64_t* rows_end, SplitFixJob* defer) {
  const BinGate gate{err, rows_end};
  if (dtype == GSGPC_F32) launch_moments_t<float>(L, p, idx, off, row0, nvalid, c_lo, c_hi, g, mom, pat, gate, sb, defer);
  else launch_moments_t<double>(L, p, idx, off, row0, nvalid, c_lo, c_hi, g, mom, pat, gate, sb, defer);
  if (nvalid > row0) L.count();
  GSGPC_CUDA(cudaGetLastError());
}

// K1p on the FP64 tensor cores (d = 3 cubic): per cell, Σ_rows s_p(row) · Π_k t_k^{e_k} is a
// GEMM over the cell's rows — A = the 64 monomials of 4 rows (8 tiles of 8), B = the ±1 signs
// of 16 probes for those rows (2 tiles of 8): 16 mma.sync.m8n8k4.f64 per 4 rows, 94 % of the
// MAC slots needed (the lane-per-probe kernel ran 64 dependent FMAs per row per lane on 8
// resident warps per SM).  Monomials are staged per row (lane) in shared memory with the
// XOR swizzle of the d = 2 K1 (conflict-free stores and fragment loads).
constexpr int PMM_PT = 2;  // probe tiles of 8 per pass

template <typename T, bool PK>
__global__ void __launch_bounds__(64) k_probe_moments_mma(RowSrc<T, PK> pay,
                                                          const uint64_t* __restrict__ pw,
                                                          const int64_t* __restrict__ off, int64_t cells,
                                                          int64_t nvalid, int64_t row0, int64_t c_lo, BinGate gate,
                                                          GridDev g, int probes, double* __restrict__ pmom,
                                                          int64_t range, int pbase, SplitRec sp) {
  constexpr int QY = 64;
  __shared__ __align__(16) double sm[2][32 * QY];
  __shared__ uint64_t swd[2][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t warp = static_cast<int64_t>(blockIdx.x) * 2 + wib;
  if (gate.closed()) return;
  sp.none(warp, lane);
  nvalid = gate.rows(nvalid);
  const int64_t r0 = row0 + warp * range;
  if (r0 >= nvalid) return;
  const int64_t rend = min(r0 + range, nvalid);
  const int nw = (probes + 63) >> 6;
  double* S = sm[wib];
  uint64_t* SW = swd[wib];
  const int r = lane >> 2, kq = lane & 3, cb = 2 * (lane & 3);
  double d[8][PMM_PT][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < PMM_PT; ++b) d[a][b][0] = d[a][b][1] = 0.0;
  int64_t c = first_cell(off, c_lo, cells, r0, lane);
  int64_t p = r0;
  bool first = true;
  while (p < rend) {
    c = next_cell(off, c, p, cells, lane);
    const int64_t ce = off[c + 1];
    const int64_t seg_end = min(ce, rend);
    double i0d[3];  // the segment's cell digits
    {
      const int64_t c12 = c / g.nc[2];
      i0d[2] = static_cast<double>(c - c12 * g.nc[2]);
      const int64_t c0 = c12 / g.nc[1];
      i0d[1] = static_cast<double>(c12 - c0 * g.nc[1]);
      i0d[0] = static_cast<double>(c0);
    }
    for (int64_t b0 = p; b0 < seg_end; b0 += 32) {
      const int nb = static_cast<int>(imin64(32, seg_end - b0));
      {
        double t[3] = {0.0, 0.0, 0.0}, y = 0.0;
        const bool v = lane < nb;
        if (v) row_t_cell<T>(g, i0d, pay[b0 + lane], t, y);
        double pk[3][4];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          double q = 1.0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            pk[k][e] = q;
            q *= t[k];
          }
        }
        double* P = S + lane * QY;
        const int sw = d2c_swz(lane);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const double ab = v ? pk[0][a] * pk[1][b] : 0.0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int q = (a * 4 + b) * 4 + e;
              P[(q & ~15) | ((q & 15) ^ sw)] = ab * pk[2][e];
            }
          }
        SW[lane] = v ? pw[pay.at(b0 + lane) * nw + (pbase >> 6)] : 0ull;
      }
      __syncwarp();
      const int steps = (nb + 3) >> 2;
      for (int st = 0; st < steps; ++st) {
        const int R = 4 * st + kq;  // rows ≥ nb were staged as zeros
        const double* P = S + R * QY;
        const int sw = d2c_swz(R);
        const uint64_t bits = SW[R];
        double bv[PMM_PT];
#pragma unroll
        for (int tb = 0; tb < PMM_PT; ++tb) {
          const int pj = (pbase & 63) + 8 * tb + r;
          bv[tb] = ((bits >> (pj & 63)) & 1ull) ? 1.0 : -1.0;
        }
#pragma unroll
        for (int ta = 0; ta < 8; ++ta) {
          const int q = 8 * ta + r;
          const double av = P[(q & ~15) | ((q & 15) ^ sw)];
#pragma unroll
          for (int tb = 0; tb < PMM_PT; ++tb) dmma(d[ta][tb][0], d[ta][tb][1], av, bv[tb]);
        }
      }
      __syncwarp();
    }
    // flush: D[r][cb + i] = monomial 8 ta + r of probe pbase + 8 tb + cb + i (split record:
    // 8·PMM_PT probes × QY per warp)
    const bool split = first && off[c] < r0;
    first = false;
#pragma unroll
    for (int ta = 0; ta < 8; ++ta)
#pragma unroll
      for (int tb = 0; tb < PMM_PT; ++tb)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int pj = pbase + 8 * tb + cb + i;
          if (pj < probes) {
            if (split) sp.v[(warp * 8 * PMM_PT + (pj - pbase)) * QY + 8 * ta + r] = d[ta][tb][i];
            else flush_val(pmom + (c * probes + pj) * QY + 8 * ta + r, d[ta][tb][i]);
          }
          d[ta][tb][i] = 0.0;
        }
    if (split && lane == 0) sp.cell[warp] = c;
    p = seg_end;
  }
}

template <typename T, bool PK>
static void launch_probe_moments(const Launch& L, const RowSrc<T, PK>& P, const uint64_t* pw, const int64_t* off,
                                 int64_t row0, int64_t nvalid, int64_t c_lo, int64_t c_hi, const GridDev& g,
                                 int probes, double* pmom, BinGate gate, const SplitBuf& sb) {
  if (nvalid <= row0) return;
  const SplitRec sp{sb.v, sb.cell};
  int QY = 1;
  for (int k = 0; k < g.d; ++k) QY *= g.W;
  const int64_t range = 1024;
  const unsigned blocks = static_cast<unsigned>(ceil_div(ceil_div(nvalid - row0, range), 2));
  static const bool lane_pm = [] {
    const char* e = getenv("GSGPC_PROBE_MOM_LANE");  // diagnostics: lane-per-probe kernel
    return e && e[0] == '1';
  }();
  if (g.d == 3 && g.W == 4 && !lane_pm) {
    const int64_t rng = 512;
    const unsigned blk = static_cast<unsigned>(ceil_div(ceil_div(nvalid - row0, rng), 2));
    if (static_cast<int64_t>(blk) * 2 > sb.warps) throw Error(GSGPC_RUNTIME_ERROR, "K1p split records undersized");
    for (int pb = 0; pb < probes; pb += 8 * PMM_PT) {
      k_probe_moments_mma<T, PK><<<blk, 64, 0, L.s>>>(P, pw, off, c_hi, nvalid, row0, c_lo, gate, g, probes, pmom, rng,
                                                   pb, sp);
      L.count();
      split_fix(L, sb, static_cast<int64_t>(blk) * 2, 8 * PMM_PT * 64, std::min(8 * PMM_PT, probes - pb) * 64, pmom,
                static_cast<int64_t>(probes) * 64, static_cast<int64_t>(pb) * 64, gate);
    }
    return;
  }
  if (static_cast<int64_t>(blocks) * 2 > sb.warps) throw Error(GSGPC_RUNTIME_ERROR, "K1p split records undersized");
  for (int pb = 0; pb < probes; pb += 32) {
#define GSGPC_PM(DD, WW)                                                                                  \
  if (g.d == DD && g.W == WW) {                                                                         \
    k_probe_moments<DD, WW, T, PK><<<blocks, 64, 0, L.s>>>(P, pw, off, c_hi, nvalid, row0, c_lo, gate, g, probes, pmom, range, pb, sp); \
  }
    GSGPC_PM(1, 2) GSGPC_PM(1, 4) GSGPC_PM(2, 2) GSGPC_PM(2, 4) GSGPC_PM(3, 2) GSGPC_PM(3, 4)
#undef GSGPC_PM
    L.count();
    split_fix(L, sb, static_cast<int64_t>(blocks) * 2, 32 * QY, std::min(32, probes - pb) * QY, pmom,
              static_cast<int64_t>(probes) * QY, static_cast<int64_t>(pb) * QY, gate);
  }
}

template <typename T>
static void launch_probe_moments_t(const Launch& L, const PointsDev& p, const int* idx, const uint64_t* pw,
                                   const int64_t* off, int64_t row0, int64_t nvalid, int64_t c_lo, int64_t c_hi,
                                   const GridDev& g, int probes, double* pmom, BinGate gate, const SplitBuf& sb) {
  if (packed4(p, g.d, sizeof(T)))
    launch_probe_moments<T, true>(L, RowSrc<T, true>{p, idx, g.d}, pw, off, row0, nvalid, c_lo, c_hi, g, probes,
                                  pmom, gate, sb);
  else
    launch_probe_moments<T, false>(L, RowSrc<T, false>{p, idx, g.d}, pw, off, row0, nvalid, c_lo, c_hi, g, probes,
                                   pmom, gate, sb);
}

void run_probe_moments(const Launch& L, int dtype, const PointsDev& p, const int* idx, const uint64_t* pw,
                       const int64_t* off, int64_t row0, int64_t nvalid, int64_t c_lo, int64_t c_hi, const GridDev& g,
                       int probes, double* pmom, const unsigned long long* err, const SplitBuf& sb,
                       const int64_t* rows_end) {
  const BinGate gate{err, rows_end};
  if (dtype == GSGPC_F32)
    launch_probe_moments_t<float>(L, p, idx, pw, off, row0, nvalid, c_lo, c_hi, g, probes, pmom, gate, sb);
  else
    launch_probe_moments_t<double>(L, p, idx, pw, off, row0, nvalid, c_lo, c_hi, g, probes, pmom, gate, sb);
  GSGPC_CUDA(cudaGetLastError());
}

// moments (cell-major [cell][QX+QY]) → stencil [S_min][m] and W^T y [m]; optional probe
// moments (cell-major [cell][P][QY]) → probe images [P][m].
void run_finalize(const Launch& L, const GridDev& g, const double* mom, int probes, const double* pmom,
                  double* stencil, double* wty, double* pimg, double* ws, int64_t ws_elems) {
  const int d = std::max(1, std::min(g.d, GSGPC_MAX_DIM)), W = g.W, E = 2 * W - 1;
  const int Q = moments_per_cell(d, W);
  int QX = 1, QY = 1;
  for (int k = 0; k < d; ++k) {
    QX *= E;
    QY *= W;
  }
  const int64_t half = ws_elems / 2;
  double* bufA = ws;
  double* bufB = ws + half;
  // chain over k = k_start .. 0.  Pass k_start reads `src`: cell-major records (stride
  // cstride, offset qoff) when cell_major, else the moment-major output of a pass over
  // k_start + 1 (ext / qext describe its extents).  Intermediates ping-pong between p0, p1.
  // outer: an untransformed leading digit of the moment index (a group of probes: the cell
  // records hold [probe][QY], the final output [probe][m]) — one launch per pass serves them all
  auto chain = [&](bool ymode, const double* src, bool cell_major, int k_start, int64_t cstride, int64_t qoff,
                   int qk0, double* final_out, int64_t c0, double* p0, double* p1, int outer = 1) {
    int64_t ext[3] = {1, 1, 1}, qext[3] = {1, 1, 1};
    for (int k = 0; k < d; ++k) {
      ext[k] = k > k_start ? g.sz[k] : g.nc[k];
      qext[k] = k > k_start ? (ymode ? 1 : E) : qk0;
    }
    const double* cur = src;
    bool first = cell_major;
    for (int k = k_start; k >= 0; --k) {
      XformDims x{};
      int64_t ext_out[3] = {1, 1, 1}, qext_out[3] = {1, 1, 1}, sp_in = 1, sp_out = 1, inner_sp = 1, inner_q = 1,
              qrest = 1;
      for (int j = 0; j < d; ++j) {
        ext_out[j] = j == k ? g.sz[k] : ext[j];
        qext_out[j] = j == k ? (ymode ? 1 : E) : qext[j];
        sp_in *= ext[j];
        sp_out *= ext_out[j];
        if (j > k) {
          inner_sp *= ext[j];
          inner_q *= qext[j];
        }
        if (j != k) qrest *= qext_out[j];
      }
      x.sp_in = static_cast<int>(sp_in);
      x.sp_out = static_cast<int>(sp_out);
      x.inner_sp = static_cast<int>(inner_sp);
      x.ext_in_k = static_cast<int>(ext[k]);
      x.ext_out_k = static_cast<int>(g.sz[k]);
      x.inner_q = static_cast<int>(inner_q);
      x.shift = W == 4 ? 1 : 0;
      x.cell_major = first ? 1 : 0;
      x.cstride = cstride;
      x.qoff = qoff;
      const bool last = k == 0;
      x.half = (last && !ymode) ? 1 : 0;
      x.c0 = c0;
      double* dst = last ? final_out : (cur == p0 ? p1 : p0);
      const dim3 grid(static_cast<unsigned>(ceil_div(sp_out, 256)), static_cast<unsigned>(qrest * outer));
      if (W == 4) {
        if (ymode) k_xform<4, true><<<grid, 256, 0, L.s>>>(cur, dst, x);
        else k_xform<4, false><<<grid, 256, 0, L.s>>>(cur, dst, x);
      } else {
        if (ymode) k_xform<2, true><<<grid, 256, 0, L.s>>>(cur, dst, x);
        else k_xform<2, false><<<grid, 256, 0, L.s>>>(cur, dst, x);
      }
      L.count();
      cur = dst;
      first = false;
      for (int j = 0; j < 3; ++j) {
        ext[j] = ext_out[j];
        qext[j] = qext_out[j];
      }
    }
  };
  const int64_t c0 = (static_cast<int64_t>(QX) - 1) / 2;
  // shared first pass (d ≥ 2): one tile of a last-dimension line staged in shared memory
  constexpr int64_t kFirstSmem = 96 * 1024;
  const int64_t rec_bytes = sizeof(double) * static_cast<int64_t>(Q);
  const int64_t max_cells = (kFirstSmem - 16) / rec_bytes;
  const int ext_out = static_cast<int>(g.sz[d - 1]);
  const int TA = static_cast<int>(std::min<int64_t>(ext_out, max_cells - (W - 1)));
  if (d >= 2 && TA >= 8) {
    XformFirst f{};
    f.Q = Q;
    f.QX = QX;
    f.ext_in = static_cast<int>(g.nc[d - 1]);
    f.ext_out = ext_out;
    int64_t lines = 1;
    for (int k = 0; k < d - 1; ++k) lines *= g.nc[k];
    f.lines = static_cast<int>(lines);
    f.TA = TA;
    f.tiles = static_cast<int>(ceil_div(ext_out, TA));
    f.qx_rest = QX / E;
    f.qy_rest = QY / W;
    f.sp_out = static_cast<int>(lines * ext_out);
    f.shift = W == 4 ? 1 : 0;
    const size_t smem = static_cast<size_t>(std::min<int64_t>(f.ext_in, TA + W - 1) * rec_bytes) + 16;
    // y intermediates live in bufB (QY·big ≤ half/2 for every (d, W) with d ≥ 2)
    double* yA = bufB;
    double* yB = bufB + half / 2;
    const unsigned blocks = static_cast<unsigned>(lines * f.tiles);
    if (W == 4) {
      set_max_dynamic_smem(reinterpret_cast<const void*>(k_xform_first<4>), static_cast<int>(kFirstSmem));
      k_xform_first<4><<<blocks, 256, smem, L.s>>>(mom, bufA, yA, f);
    } else {
      set_max_dynamic_smem(reinterpret_cast<const void*>(k_xform_first<2>), static_cast<int>(kFirstSmem));
      k_xform_first<2><<<blocks, 256, smem, L.s>>>(mom, bufA, yA, f);
    }
    L.count();
    chain(true, yA, false, d - 2, 0, 0, W, wty, 0, yB, yA);
    chain(false, bufA, false, d - 2, 0, 0, E, stencil, c0, bufB, bufA);
  } else {
    chain(true, mom, true, d - 1, Q, QX, W, wty, 0, bufA, bufB);
    chain(false, mom, true, d - 1, Q, 0, E, stencil, c0, bufA, bufB);
  }
  // probe images: groups of probes per pass (the largest y intermediate of a probe is
  // QY/W · max(m, cells) doubles; a group fills one ping-pong buffer).  One probe per chain,
  // reading its QY values at a P·QY stride between cells, took 8.8 ms at config 5 (30 probes).
  if (pmom != nullptr && probes > 0) {
    const int64_t inter = static_cast<int64_t>(QY / W) * std::max(g.m, g.cells);
    const int grp = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(probes, half / std::max<int64_t>(inter, 1))));
    for (int pj = 0; pj < probes; pj += grp) {
      const int ng = std::min(grp, probes - pj);
      chain(true, pmom, true, d - 1, static_cast<int64_t>(probes) * QY, static_cast<int64_t>(pj) * QY, W,
            pimg + static_cast<int64_t>(pj) * g.m, 0, bufA, bufB, ng);
    }
  }
  GSGPC_CUDA(cudaGetLastError());
}

int64_t finalize_ws_elems(const GridDev& g) {
  const int W = g.W, E = 2 * W - 1;
  int64_t QX = 1, QY = 1;
  for (int k = 0; k < g.d; ++k) {
    QX *= E;
    QY *= W;
  }
  const int64_t big = std::max(g.m, g.cells);
  return 2 * std::max(QX, QY) * big;  // two ping-pong buffers of the largest intermediate
}

// ------------------------------------------------------------------ W^T W structure (export)
// touched[s][a] = 1 iff some row gave nonzero weights to both node a and node a + o_s: a cell
// whose stencil covers both and one of its zero-weight patterns (see pat_bit) keeps both
// slots nonzero in every dimension.
__global__ void k_touched(GridDev g, int64_t total, const uint8_t* __restrict__ pat, uint8_t* __restrict__ out) {
  const int W = g.W, E = 2 * W - 1, o = W / 2 - 1;
  int S = 1, P = 1;
  for (int k = 0; k < g.d; ++k) {
    S *= E;
    P *= 3;
  }
  const int c0 = (S - 1) / 2;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int s = static_cast<int>(idx / g.m);
    int64_t a = idx - static_cast<int64_t>(s) * g.m;
    int q = c0 + s;
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, ak[3] = {0, 0, 0}, dk[3] = {0, 0, 0};
    bool ok = true;
    for (int k = g.d - 1; k >= 0; --k) {
      dk[k] = q % E - (W - 1);
      q /= E;
      ak[k] = static_cast<int>(a % g.sz[k]);
      a /= g.sz[k];
      const int b = ak[k] + dk[k];
      if (b < 0 || b >= g.sz[k]) ok = false;
      lo[k] = max(max(ak[k], b) - (W - 1 - o), 0);
      hi[k] = min(min(ak[k], b) + o, static_cast<int>(g.nc[k]) - 1);
      if (lo[k] > hi[k]) ok = false;
    }
    bool hit = false;
    if (ok) {
      for (int i0 = lo[0]; i0 <= hi[0] && !hit; ++i0)
        for (int i1 = g.d > 1 ? lo[1] : 0; i1 <= (g.d > 1 ? hi[1] : 0) && !hit; ++i1)
          for (int i2 = g.d > 2 ? lo[2] : 0; i2 <= (g.d > 2 ? hi[2] : 0) && !hit; ++i2) {
            const int ic[3] = {i0, i1, i2};
            int64_t cell = 0;
            int allow[3] = {1, 1, 1};  // bit j: pattern j allowed in dimension k
            for (int k = 0; k < g.d; ++k) {
              cell = cell * g.nc[k] + ic[k];
              const int sa = ak[k] - ic[k] + o;
              if (dk[k] == 0 && sa == o) allow[k] |= 2;
              if (dk[k] == 0 && sa == o + 1) allow[k] |= 4;
            }
            const uint8_t* pc = pat + cell * P;
            for (int p = 0; p < P && !hit; ++p) {
              int r = p;
              bool al = true;
              for (int k = 0; k < g.d; ++k) {
                al = al && ((allow[k] >> (r % 3)) & 1);
                r /= 3;
              }
              hit = al && pc[p] != 0;
            }
          }
    }
    out[idx] = hit ? 1 : 0;
  }
}

void run_touched(const Launch& L, const GridDev& g, int S_min, const uint8_t* pat, uint8_t* out) {
  const int64_t total = static_cast<int64_t>(S_min) * g.m;
  const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), sm_count() * 16)));
  k_touched<<<blocks, 256, 0, L.s>>>(g, total, pat, out);
  L.count();
  GSGPC_CUDA(cudaGetLastError());
}

__global__ void k_or_bytes(int64_t n, uint8_t* __restrict__ dst, const uint8_t* __restrict__ src) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] |= src[i];
}

void run_or_bytes(const Launch& L, int64_t n, uint8_t* dst, const uint8_t* src) {
  if (n <= 0) return;
  const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), sm_count() * 8)));
  k_or_bytes<<<blocks, 256, 0, L.s>>>(n, dst, src);
  L.count();
  GSGPC_CUDA(cudaGetLastError());
}

}  // namespace gsgpc

