// precompute.cuh — host entry points of the kernels in precompute.cu / operators.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <memory>
#include <utility>
#include <vector>

#include "internal.cuh"

namespace gsgpc {

// Stream + launch counter (every library kernel launch is counted: gsgpc_ctx_launch_count).
// GSGPC_DEBUG_SYNC=1 (diagnostics): synchronize after every counted launch and report the
// first failing one by its ordinal.
bool debug_sync_enabled();
void debug_sync_check(cudaStream_t s, uint64_t ordinal);
struct Launch {
  cudaStream_t s;
  uint64_t* counter;
  void count(int k = 1) const {
    *counter += static_cast<uint64_t>(k);
    if (debug_sync_enabled()) debug_sync_check(s, *counter);
  }
};

// ---- precompute.cu
int moments_per_cell(int d, int W);
int64_t finalize_ws_elems(const GridDev& g);
// Binning (two-level counting sort, see precompute.cu K2): bucket = cell >> bsh.
struct BinDesc {
  int bsh, nb;
};
BinDesc bin_desc(int64_t cells);
int64_t bin_tiles(int64_t n);   // rows per tile: TILE_ROWS
int64_t bin_groups(int64_t n);  // tile groups of the tile scan
void run_classify(const Launch& L, int dtype, const PointsDev& p, int64_t n, int64_t row0, const GridDev& g,
                  const BinDesc& bd, int* tcnt, unsigned long long* err, double* part, int nblk, int* cellid);
void run_sum_partials(const Launch& L, const double* part, int np, double* acc);
// bucket sizes: bbase[nb + 1] (row offsets), sbase[nb + 1] (slice offsets); gsum scratch [groups][nb]
// bucket totals → bbase / sbase; tcnt (per-tile bucket counts) becomes the per-tile output
// offsets the partition places each tile's runs at (row order: deterministic)
void run_bucket_totals(const Launch& L, const BinDesc& bd, int64_t n, int* tcnt, int* gsum, int64_t* bbase,
                       int64_t* sbase);
int64_t bin_slices_max(int64_t nvalid, const BinDesc& bd);
// keys (cellid[i], i) → bucket-contiguous cid1 / idx1, in a fixed order within each bucket
// (toff: the per-tile offsets from run_bucket_totals).  The rows themselves never move: K1
// gathers them through the sorted indices.
// Kernels that commit take the device error word of the classify pass (err) and return at
// once when it records an out-of-grid row; rows_end (device) bounds the rows binned.
void run_partition(const Launch& L, int64_t n, const BinDesc& bd, const int* cellid, const int* toff, int* cid1,
                   int* idx1, const unsigned long long* err);
// dst += src unless err records an error
void run_commit_add(const Launch& L, const unsigned long long* err, const double* src, double* dst);
// bucket-contiguous keys → cell-sorted row indices idx_s and off[] for buckets [b0, b1) =
// slices [s0, s1) (off[cells] written by the last bucket); scnt: slices × 2^bsh
void run_slice_sort(const Launch& L, const BinDesc& bd, int64_t cells, int b0, int b1, int64_t s0, int64_t s1,
                    const int* cid1, const int* idx1, const int64_t* bbase, const int64_t* sbase, int* scnt,
                    int64_t* off, int* idx_s, const unsigned long long* err);
// K1 split records (bitwise-reproducible flushes of cells split across warp ranges, see
// precompute.cu SplitRec): device scratch of warps × rec doubles + warps int64
struct SplitBuf {
  double* v;
  int64_t* cell;
  int64_t warps;
  int64_t rec;
};
int64_t split_rec_warps(int64_t rows);
int64_t split_rec_doubles(const GridDev& g, int probes);
// The split-record fix-up of a K1 launch (adds the partials of cells continued across warp
// ranges, in warp order).  run_moments runs it itself unless asked to hand it back.
struct SplitFixJob {
  int64_t nwarps;
  int rec, qv;
  double* M;
  int64_t mstride, mbase;
  const unsigned long long* err;
  const int64_t* rows_end;
  bool pending;
};
void run_split_fix(const Launch& L, const SplitBuf& sb, const SplitFixJob& job);
// K1 over sorted rows [row0, nvalid) whose cells lie in [c_lo, c_hi) (off[] read only there);
// sorted row p is batch row idx[p] of p (the batch's points, as classified).  defer: the split
// fix-up is returned there instead of launched (the caller runs run_split_fix before the next
// K1 launch that uses the same split records).
void run_moments(const Launch& L, int dtype, const PointsDev& p, const int* idx, const int64_t* off, int64_t row0,
                 int64_t nvalid, int64_t c_lo, int64_t c_hi, const GridDev& g, double* mom, uint8_t* pat,
                 const unsigned long long* err, const SplitBuf& sb, const int64_t* rows_end = nullptr,
                 SplitFixJob* defer = nullptr);
// probe words pw: [batch row][⌈P/64⌉] (bit j of word w: probe 64w + j is +1)
void run_probe_moments(const Launch& L, int dtype, const PointsDev& p, const int* idx, const uint64_t* pw,
                       const int64_t* off, int64_t row0, int64_t nvalid, int64_t c_lo, int64_t c_hi, const GridDev& g,
                       int probes, double* pmom, const unsigned long long* err, const SplitBuf& sb,
                       const int64_t* rows_end = nullptr);
// W^T W structure: touched[S_min][m] (0/1) from the per-cell zero-weight patterns
// (cells × 3^d bytes written by K1); byte-wise OR for merges.
void run_touched(const Launch& L, const GridDev& g, int S_min, const uint8_t* pat, uint8_t* out);
void run_or_bytes(const Launch& L, int64_t n, uint8_t* dst, const uint8_t* src);

void run_finalize(const Launch& L, const GridDev& g, const double* mom, int probes, const double* pmom,
                  double* stencil, double* wty, double* pimg, double* ws, int64_t ws_elems);

// ---- operators.cu
// Symmetric half stencil: offsets s = 0..S_min-1 (lexicographically non-negative), per-dim
// displacements in [-(W-1), W-1].
struct StencilDesc {
  int d, W, S_min;
  int64_t sz[GSGPC_MAX_DIM];
  int64_t m;
};
// Stencil offset tables.  Kernels receive them BY VALUE as __grid_constant__ parameters (the
// launch's own constant bank, read like __constant__ memory): no module-global table that two
// contexts, streams or threads could overwrite under each other's in-flight kernels.
constexpr int kMaxSmin = 172;  // (7^3 + 1) / 2
constexpr int kMaxPen = 49;    // 7^2 pencils along the last dimension
struct StencilOffsets {
  long long flat[kMaxSmin];     // flat offset o_s of half-stencil entry s
  int o32[kMaxSmin];            // the same in 32 bits (S_min·m < 2^31 checked by the callers)
  signed char d[kMaxSmin][4];   // per-dimension displacements
};
struct PencilTables {           // the full stencil as E^(d−1) pencils along the last dimension
  int ob[kMaxPen];              // base flat offset of pencil q (last digit 0)
  int s[kMaxPen][7];            // per last-dimension shift: half index (≥ 0) or −(index + 1) (mirrored)
};
StencilOffsets make_stencil_offsets(const StencilDesc& sd);
PencilTables make_pencil_tables(const StencilDesc& sd);
// out = (W^T W) v ; if dot_out != nullptr also dot(out, dotv) via deterministic partials.
// flag (optional, device int): set to 1 when some row's sum is not finite (see k_spmv)
void run_spmv(const Launch& L, const StencilDesc& sd, const double* A, const double* v, double* out,
              int* flag = nullptr);
// recompute the non-finite rows of out over the touched pairs only (touched: [S_min][m] bytes)
void run_spmv_touched(const Launch& L, const StencilDesc& sd, const double* A, const double* v,
                      const uint8_t* touched, double* out);

// Kronecker K_G (Toeplitz mode products)
struct KgFft;  // operators.cu: circulant-embedding FFT route for large dimensions
struct KgDev {
  int d;
  int64_t sz[GSGPC_MAX_DIM];
  int64_t m;
  const double* gen[GSGPC_MAX_DIM];  // per-dim generator columns (outputscale folded into dim 0)
  KgFft* fft;                        // host object (never read on the device); nullptr: no FFT dims
};
// next_fast_fft_size (grid.cpp:73-82): smallest 5-smooth integer ≥ x
int64_t next_fast_fft_size(int64_t x);
// default: dimensions with more nodes than the tensor-core mode products hold (2040) take the
// circulant FFT route
constexpr int64_t kKgFftMinNodes = 2041;
// Builds the FFT route for the dimensions of kg with ≥ min_nodes nodes (nullptr if none):
// per dimension the spectrum of T_k's circulant embedding (size next_fast_fft_size(2 n_k − 1),
// grid.cpp:94-151 restricted to one factor of the separable kernel) and cuFFT plans for one
// m-vector.  Synchronises the stream.
std::shared_ptr<KgFft> kg_fft_create(const KgDev& kg, int64_t min_nodes, cudaStream_t s);
bool kg_fft_dim(const KgDev& kg, int k);
void run_kg_apply(const Launch& L, const KgDev& kg, const double* v, double* out, double* tmp0, double* tmp1);
// `batch` contiguous m-vectors at once (tmp0 / tmp1 hold batch·m doubles)
void run_kg_apply_batched(const Launch& L, const KgDev& kg, int64_t batch, const double* v, double* out,
                          double* tmp0, double* tmp1);

// EFCG (see operators.cu)
struct CgState {
  double rho, rho_new, pap, alpha, beta, eps, eps_abs, rel_tol, sigma_sq;
  int iter, maxiter, done, converged, breakdown;
  unsigned int cnt_a, cnt_b;
};
struct CgBufs {
  double *r, *u, *s, *z, *x;     // rhat, uhat, shat, zbar, xhat_d
  double *kt0, *kt1;             // K_G temporaries
  double *part_a, *part_b;       // block partials for the two dots
  double *trace, *alphas, *betas;
  CgState* st;
};
void run_cg_init(const Launch& L, const StencilDesc& sd, const double* A, const KgDev& kg, const CgBufs& b,
                 int64_t m);
void run_cg_iter(const Launch& L, const StencilDesc& sd, const double* A, const KgDev& kg, const CgBufs& b,
                 int64_t m);
int cg_partials_needed(int64_t m);
// efcg_persistent.cu: the whole solve in one cooperative launch (init = run the r̂0 setup first)
void run_efcg_persistent(const Launch& L, const StencilDesc& sd, const double* A, const KgDev& kg, const CgBufs& b,
                         int init, unsigned long long* tbuf = nullptr);

// Vector helpers
void run_axpby(const Launch& L, int64_t n, double a, const double* x, double b, const double* y, double* out);
void run_scale(const Launch& L, int64_t n, double a, const double* x, double* out);

// Point-wise interpolation (bit-exact weights)
void run_interp_weights(const Launch& L, int dtype, const PointsDev& p, int64_t n, const GridDev& g,
                        int64_t* idx, double* w, int* nnz, int* status);
void run_predict(const Launch& L, int dtype, const PointsDev& p, int64_t n, const GridDev& g, const double* coeffs,
                 double* out, int* status);

// ---- efla.cu: probe-batched EFLA (P <= 32 per call; inputs device arrays P × m)
struct EflaOut {
  std::vector<double> alpha, beta, d;  // P × k
  std::vector<int> order;
};
// basis_out (optional, device P × k × m): the Q̂ columns (TridiagonalFactor::basis)
EflaOut efla_run(const Launch& L, const StencilDesc& sd, const double* A, const KgDev& kg, int P, const double* kwt_in,
                 const double* wt_in, const double* z0sq_dev, double s2, int k, double* basis_out = nullptr);
std::pair<double, int> quadrature_logdet_host(const double* alpha, const double* beta, int k, double probe_sq,
                                              double quad_tol);
void run_kg_batched(const Launch& L, const KgDev& kg, int P, const double* v, double* out, double* t0, double* t1);
// plain batched Lanczos (solvers.cpp:351-389) and the SymmetricGrid / Dense log-det routes
struct LanczosOut {
  std::vector<double> alpha, beta;  // P × k
  std::vector<int> order;
};
using BatchedOp = std::function<void(const double* in, double* out)>;
LanczosOut lanczos_batched(const Launch& L, int64_t m, int P, int k, const double* start, const BatchedOp& op);
double slq_logdet_sum(const Launch& L, int64_t m, int p_begin, int p_end, int max_depth, double quad_tol,
                      uint64_t seed, const std::function<BatchedOp(int)>& make_op);
BatchedOp kg_op(const Launch& L, const KgDev& kg, int P, double* t0, double* t1);
BatchedOp sym_op(const Launch& L, const StencilDesc& sd, const double* A, const KgDev& kg, int P, double sigma_sq,
                 double* ku, double* wku, double* t0, double* t1);
double kg_condition_estimate(const Launch& L, const KgDev& kg);
double dense_logdet_grid_system(const Launch& L, const StencilDesc& sd, const double* A, const KgDev& kg,
                                double sigma_sq);
// multi-RHS EFCG (P ≤ 32 per call): x (P × m, device) ← x̂_d of each RHS
struct BcgOut {
  std::vector<int> iterations, converged;
  std::vector<double> residual_sq;
  bool breakdown = false;
};
BcgOut bcg_run(const Launch& L, const StencilDesc& sd, const double* A, const KgDev& kg, int P, const double* rhat0,
               double sigma, double eps_abs, double rel_tol, int maxiter, double* x);
// covariance helpers (device, row-major)
void cov_scatter_w(const Launch& L, int64_t ns, int64_t m, int cap, const int64_t* idx, const double* w,
                   const int* nnz, double* out);
void cov_gather(const Launch& L, int64_t ni, int64_t nh, int64_t m, int cap, const int64_t* idx, const double* w,
                const int* nnz, const double* H, double* out);
void cov_sub_abt(const Launch& L, int n, int64_t m, const double* A, const double* B, double* C);
void spmm_batched(const Launch& L, const StencilDesc& sd, const double* A, const double* x, double* out, int P);

// ---- probe_rng.cu: rademacher_probe streams (std::mt19937_64 per probe) on the device
void mt_seed_state(uint64_t seed, uint64_t p, uint64_t* st /*313*/);
// substream starts are multiples of kJumpUnit blocks of 312 draws (mt_jump.cu caches the
// jump polynomials of those multiples)
constexpr uint64_t kJumpUnit = 3360;
int64_t probe_rng_slab(int P);
int64_t probe_rng_scratch_words(int P);
// next `rows` draws of every probe: states P × 313 (device), planes ≥ P × slab bytes scratch,
// words[rows] (bit p = probe p is +1), scratch ≥ probe_rng_scratch_words(P) device words
void run_probe_rng(const Launch& L, uint64_t* states, int P, int64_t rows, uint8_t* planes, uint64_t* words,
                   uint64_t* scratch);
// ---- mt_jump.cu: GF(2) jump-ahead of the MT19937-64 streams
// out[s·K + k] = stream s (in: S × 313, window + index) advanced by 312·q[k] draws; polys_dev
// ≥ K × 312 device words of scratch.  Synchronises the stream (host staging).
void run_mt_jump(const Launch& L, const uint64_t* in, int S, const std::vector<uint64_t>& q, uint64_t* polys_dev,
                 uint64_t* out);
// host restatement: st (313 words) advanced by `draws` draws
void mt_jump_host(uint64_t* st, uint64_t draws);

}  // namespace gsgpc
