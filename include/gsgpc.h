/*
 * gsgpc.h — C ABI of the B200-native GSGP hot path (libgsgpc.so).
 *
 * Drop-in boundary for the reference's proj/include/gsgp C++ API
 * (/root/reference/proj/include/gsgp/{interp,grid,solvers,gp,io}.hpp).  Each entry point
 * names the reference interface it replaces (file:line).  Plain pointers and sizes only:
 * no torch, no Eigen, no exceptions cross this boundary.
 *
 * Memory: every `const double* / double*` array argument may live in host memory
 * (pageable or pinned) or in device memory of the context's GPU; the library detects
 * which (cudaPointerGetAttributes) and stages host arrays through the context's stream.
 * Handles own their device buffers; callers own their arrays.
 *
 * Errors: functions return a gsgpc_status; gsgpc_last_error(ctx) holds the reference's
 * message text ("sufficient_stats: stream row 17: interp_weights: point outside grid",
 * "factorized_cg_grid_rhs: p^T A p <= 0, ...").  OUT_OF_GRID also records the 1-based
 * minimum offending row (gsgpc_last_error_row), i.e. the row at which the reference's
 * single pass would have thrown.  A failed call leaves its handles unchanged.
 *
 * Threading: one CUDA stream per context; calls on one context are serialised by the
 * caller (the C++/Python wrappers do this).  Device-resident inputs are read on the
 * context's stream (gsgpc_ctx_stream / gsgpc_ctx_set_stream): the caller orders their
 * producers before the call (the Python mirror waits for torch's current stream), and
 * device-resident outputs are complete once the context's stream is.  Contexts on different devices are
 * independent; multi-GPU precompute combines per-device statistics with an all-reduce
 * over gsgpc_stats_reduce_buffer() (merge() semantics, interp.cpp:202-210).
 */
#ifndef GSGPC_H
#define GSGPC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSGPC_MAX_DIM 3

typedef enum {
  GSGPC_OK = 0,
  GSGPC_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  GSGPC_OUT_OF_GRID = 2,      /* std::invalid_argument from interp_weights (interp.cpp:53-55,119-124) */
  GSGPC_BREAKDOWN = 3,        /* SolverBreakdown (solvers.hpp:73-76) */
  GSGPC_NONCONVERGENCE = 4,   /* SolverNonConvergence (gp.hpp:17-23) */
  GSGPC_CUDA_ERROR = 5,
  GSGPC_UNSUPPORTED = 6,      /* valid for the reference, outside this build (e.g. d > 3) */
  GSGPC_RUNTIME_ERROR = 7,    /* std::runtime_error (negative Ritz value, gp.cpp:44-47) */
} gsgpc_status;

/* InterpScheme (interp.hpp:15); the numeric values match the stats-file encoding
 * (io.cpp:205: 0 = Linear, 1 = Cubic). */
typedef enum { GSGPC_LINEAR = 0, GSGPC_CUBIC = 1 } gsgpc_scheme;

typedef enum { GSGPC_F32 = 0, GSGPC_F64 = 1 } gsgpc_dtype;

typedef struct gsgpc_ctx gsgpc_ctx;
typedef struct gsgpc_stats gsgpc_stats;
typedef struct gsgpc_kg gsgpc_kg;

/* gsgp::Grid / GridDim (grid.hpp:15-44): row-major flattening, last dimension fastest. */
typedef struct {
  int32_t dim;
  double min[GSGPC_MAX_DIM];
  double max[GSGPC_MAX_DIM];
  int64_t size[GSGPC_MAX_DIM];
} gsgpc_grid;

/* A batch of data rows — the RowStream::next (interp.hpp:150-155) source, in memory.
 * Coordinate k of row i is at  x[i*x_row_stride + x_col_offset[k]],  the response at
 * y[i*y_stride]  (element units of `dtype`).  Covers SoA, AoS (x..., y) rows such as the
 * reference's GSGPDAT1 f64 rows (io.hpp:31-45), and packed fp32 float4 (x1,x2,x3,y). */
typedef struct {
  int32_t dtype; /* gsgpc_dtype, shared by x and y */
  const void* x;
  int64_t x_row_stride;
  int64_t x_col_offset[GSGPC_MAX_DIM];
  const void* y;
  int64_t y_stride;
} gsgpc_points;

/* ---------------------------------------------------------------- context */
gsgpc_status gsgpc_ctx_create(int device, gsgpc_ctx** out);
/* Several GPUs from one process (SURVEY §8(b) gsgpc_ctx_create(device_ids[], ngpu)): one
 * context per listed device plus, for distinct devices, an NCCL communicator over them
 * (libnccl resolved at run time; a group listing a device twice exchanges through peer
 * copies).  gsgpc_group_ctx(g, r) is device r's context (owned by the group). */
typedef struct gsgpc_group gsgpc_group;
gsgpc_status gsgpc_group_create(const int* device_ids, int ngpu, gsgpc_group** out);
gsgpc_status gsgpc_group_destroy(gsgpc_group* group);
gsgpc_status gsgpc_group_info(const gsgpc_group* group, int* ngpu, int* uses_nccl);
gsgpc_ctx* gsgpc_group_ctx(gsgpc_group* group, int rank);
const char* gsgpc_group_last_error(const gsgpc_group* group);
int64_t gsgpc_group_last_error_row(const gsgpc_group* group);
void gsgpc_ctx_destroy(gsgpc_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL restores the own one. */
gsgpc_status gsgpc_ctx_set_stream(gsgpc_ctx* ctx, void* cuda_stream);
void* gsgpc_ctx_stream(gsgpc_ctx* ctx);
gsgpc_status gsgpc_ctx_synchronize(gsgpc_ctx* ctx);
const char* gsgpc_last_error(const gsgpc_ctx* ctx);
int64_t gsgpc_last_error_row(const gsgpc_ctx* ctx);
/* Number of library kernels launched on this context so far (instrumentation). */
uint64_t gsgpc_ctx_launch_count(const gsgpc_ctx* ctx);
/* Per-phase device timing (CUDA events on the context stream), off by default.
 * Phases: 0 classify/count, 1 scan, 2 scatter, 3 moments (K1), 4 finalize, 5 H2D, 6 K1 split
 * fix-up, 7 probe moments, 8 probe streams (device MT19937-64), 9 reserved. */
gsgpc_status gsgpc_ctx_enable_phase_timing(gsgpc_ctx* ctx, int enable);
gsgpc_status gsgpc_ctx_phase_times(gsgpc_ctx* ctx, double* ms_out /*[10]*/, int64_t* calls_out /*[10]*/);
gsgpc_status gsgpc_ctx_reset_phase_times(gsgpc_ctx* ctx);
/* Diagnostics: measured FP64 FMA throughput of this GPU (TFLOP/s, 2 flops per DFMA) from a
 * register-resident DFMA loop over all SMs — the denominator of the precompute's FP64 roofline. */
gsgpc_status gsgpc_diag_fp64_peak(gsgpc_ctx* ctx, double* tflops);
/* Diagnostics: FP64 tensor-core (mma.sync m8n8k4 f64) throughput, alone and interleaved
 * with DFMA chains in the same warps (TFLOP/s). */
gsgpc_status gsgpc_diag_fp64_tensor(gsgpc_ctx* ctx, double* dmma_tflops, double* mixed_tflops);
/* Library build identification ("gsgpc sm_100a <git> ..."). */
const char* gsgpc_version(void);

/* ---------------------------------------------------------------- grid helpers */
/* fit_grid_to_data (interp.hpp:168-172, interp.cpp:286-306). */
gsgpc_status gsgpc_fit_grid_to_data(int dim, const double* lo, const double* hi,
                                    const int64_t* sizes, int scheme, gsgpc_grid* out);

/* interp_weights (interp.hpp:38-41, interp.cpp:79-134) for n points, bit-exact: idx/w are
 * n × (2r)^d (row i holds nnz[i] entries in the reference's order, exact zeros dropped);
 * status[i] = 0 ok, 1 point outside grid, 2 stencil leaves the grid. Arrays host or device. */
gsgpc_status gsgpc_interp_weights(gsgpc_ctx* ctx, const gsgpc_grid* grid, int scheme,
                                  const gsgpc_points* pts, int64_t n, int64_t* idx, double* w,
                                  int32_t* nnz, int32_t* status);

/* ---------------------------------------------------------------- sufficient statistics */
/* SufficientStatsAccumulator(Grid, InterpScheme) (interp.hpp:87-91, interp.cpp:179-186). */
gsgpc_status gsgpc_stats_create(gsgpc_ctx* ctx, const gsgpc_grid* grid, int scheme,
                                gsgpc_stats** out);
void gsgpc_stats_destroy(gsgpc_stats* stats);
/* SufficientStatsAccumulator::add over a batch of n rows (interp.cpp:188-200), rows
 * numbered after the rows already added.  Optional probe_words (n × ceil(P/64) uint64, bit p of
 * row i = sign of the p-th Rademacher probe, +1 when set) accumulate the probe images W^T v_p
 * used by the factorized SLQ (gp.cpp:97-99); pass NULL / 0 otherwise. */
gsgpc_status gsgpc_stats_add(gsgpc_ctx* ctx, gsgpc_stats* stats, const gsgpc_points* pts,
                             int64_t n, const uint64_t* probe_words, int probes);
/* Accumulate every row of a GSGPDAT1 dataset file (BinaryRowStream, io.hpp:31-45,
 * io.cpp:103-122: magic "GSGPDAT1", u64 n, u64 d, n rows of (d+1) little-endian f64) —
 * sufficient_stats(grid, scheme, BinaryRowStream(path)) (interp.cpp:244-263) when stats is
 * fresh.  Reading, host-to-device copies and the precompute overlap (pinned double buffers).
 * Errors as the reference: "cannot open binary dataset", "bad magic in binary dataset",
 * "truncated file while reading row count|dimension|coordinate|response", "binary dataset:
 * bad dimension", "sufficient_stats: stream/grid dimension mismatch", and
 * GSGPC_OUT_OF_GRID "sufficient_stats: stream row N: ..." with N counted from the file's
 * first row.  On error the accumulator is unchanged.  rows_added may be NULL. */
gsgpc_status gsgpc_stats_add_file(gsgpc_ctx* ctx, gsgpc_stats* stats, const char* path, int64_t* rows_added);
/* Accumulate probe images of the reference's Rademacher probes (rademacher_probe,
 * gp.cpp:16-25: std::seed_seq{seed_lo, seed_hi, p_lo, p_hi} + std::mt19937_64, one draw per
 * row in stream order) for p = 0..probes-1 in every following gsgpc_stats_add; the library
 * generates the streams itself on the device (one block per probe and substream), continuing
 * across batches.  Call before the first row is added.  probes <= 64. */
gsgpc_status gsgpc_stats_enable_probes(gsgpc_ctx* ctx, gsgpc_stats* stats, int probes, uint64_t seed);
/* The same streams positioned at draw `first_row`: for an accumulator (a rank's shard) whose
 * rows are rows [first_row, first_row + n) of one global stream, so that shard probe images
 * sum (merge / all-reduce) to the single-pass W^T v_p of rademacher_probe over the whole
 * stream.  The streams are advanced by GF(2) jump-ahead (no draws are generated).  merge()
 * of probe-seeded shards requires adjacent row ranges. */
gsgpc_status gsgpc_stats_enable_probes_at(gsgpc_ctx* ctx, gsgpc_stats* stats, int probes, uint64_t seed,
                                          int64_t first_row);
/* Test hook (host only, needs no GPU): bit 0 of draws [offset, offset + n) of
 * rademacher_probe's stream for (seed, p) (gp.cpp:16-25), reached by the library's jump-ahead
 * (out[i] = 1 ↔ +1). */
gsgpc_status gsgpc_probe_stream_bits(uint64_t seed, uint64_t p, uint64_t offset, int64_t n, uint8_t* out);
/* Reset an accumulator to the freshly constructed state (no rows), keeping its buffers —
 * equivalent to constructing a new SufficientStatsAccumulator on the same grid. */
gsgpc_status gsgpc_stats_reset(gsgpc_ctx* ctx, gsgpc_stats* stats);
/* SufficientStatsAccumulator::merge (interp.cpp:202-210): dst += src (same device). */
gsgpc_status gsgpc_stats_merge(gsgpc_ctx* ctx, gsgpc_stats* dst, const gsgpc_stats* src);
/* SufficientStatsAccumulator::finalize (interp.cpp:212-221): cell moments → W^T W stencil,
 * W^T y.  Called implicitly by every consumer below. */
gsgpc_status gsgpc_stats_finalize(gsgpc_ctx* ctx, gsgpc_stats* stats);
/* sufficient_stats (interp.hpp:159-160, interp.cpp:244-263): create + add + finalize. */
gsgpc_status gsgpc_sufficient_stats(gsgpc_ctx* ctx, const gsgpc_grid* grid, int scheme,
                                    const gsgpc_points* pts, int64_t n, gsgpc_stats** out);

/* SufficientStats accessors (interp.hpp:128-146): grid_size() m, n(), yty(), and the
 * stored W^T W layout: n_offsets = (S+1)/2 symmetric stencil offsets, S = (4r-1)^d. */
gsgpc_status gsgpc_stats_info(gsgpc_ctx* ctx, gsgpc_stats* stats, int64_t* m, int64_t* n,
                              double* yty, int64_t* n_offsets, int32_t* probes);
gsgpc_status gsgpc_stats_grid(const gsgpc_stats* stats, gsgpc_grid* grid, int* scheme);
/* W^T y (m doubles). */
gsgpc_status gsgpc_stats_copy_wty(gsgpc_ctx* ctx, gsgpc_stats* stats, double* out);
/* W^T W as the symmetric stencil: values n_offsets × m (offset-major), offsets n_offsets × dim
 * integer displacements (lexicographically non-negative half, offset 0 first). */
gsgpc_status gsgpc_stats_copy_stencil(gsgpc_ctx* ctx, gsgpc_stats* stats, double* values,
                                      int32_t* offsets);
/* Probe images W^T v_p (probes × m) accumulated by gsgpc_stats_add. */
gsgpc_status gsgpc_stats_copy_probe_images(gsgpc_ctx* ctx, gsgpc_stats* stats, double* out);
/* SufficientStats::wtw() as RowMajor CSR (interp.hpp:129): exact zeros are not stored,
 * columns ascending.  nnz first (values may be NULL), then fill host arrays. */
gsgpc_status gsgpc_stats_csr_nnz(gsgpc_ctx* ctx, gsgpc_stats* stats, int64_t* nnz,
                                 int64_t* max_row_nnz);
gsgpc_status gsgpc_stats_export_csr(gsgpc_ctx* ctx, gsgpc_stats* stats, int64_t* row_ptr,
                                    int64_t* col, double* val);
/* SufficientStats::apply_wtw (interp.hpp:135-136, interp.cpp:227-233). */
gsgpc_status gsgpc_stats_apply_wtw(gsgpc_ctx* ctx, gsgpc_stats* stats, const double* v,
                                   double* out);
/* Contiguous device buffer [stencil | W^T y | probe images | yty | n] of a finalized
 * stats object, for an in-place sum all-reduce across ranks (NCCL via torch.distributed);
 * call gsgpc_stats_mark_reduced() afterwards (the object then accepts no more add()). */
gsgpc_status gsgpc_stats_reduce_buffer(gsgpc_ctx* ctx, gsgpc_stats* stats, double** dev_ptr,
                                       int64_t* count);
/* Device bytes (cells x 3^d, 0/1) recording which zero-weight patterns each cell's rows had:
 * the structure of W^T W (the reference's hash keys, interp.cpp:188-200), kept apart from
 * the values.  Ranks combine them with an in-place MAX all-reduce (= OR) before
 * gsgpc_stats_mark_reduced(). */
gsgpc_status gsgpc_stats_pattern_buffer(gsgpc_ctx* ctx, gsgpc_stats* stats, uint8_t** dev_ptr,
                                        int64_t* count);
gsgpc_status gsgpc_stats_mark_reduced(gsgpc_ctx* ctx, gsgpc_stats* stats);
/* sufficient_stats (interp.cpp:244-263) sharded over a group's devices: device r takes rows
 * [r*n/G, (r+1)*n/G) of pts (host or device memory), the shards' statistics are finalized and
 * combined with one all-reduce — merge() semantics (interp.cpp:202-210): W^T W, W^T y, yty, n
 * summed, W^T W structure united — so out[r] (device r) each hold the full statistics.
 * probes > 0: Rademacher probe images with the reference's streams (gp.cpp:16-25), each shard
 * starting its streams at its first row.  OUT_OF_GRID reports the first bad row of the whole
 * batch (gsgpc_group_last_error_row).  out: ngpu handles. */
gsgpc_status gsgpc_group_sufficient_stats(gsgpc_group* group, const gsgpc_grid* grid, int scheme,
                                          const gsgpc_points* pts, int64_t n, int probes, uint64_t seed,
                                          gsgpc_stats** out);
/* The exchange step alone: stats[r] (finalized, on device r, same grid and scheme) become their
 * sum (merge(), interp.cpp:202-210) on every device. */
gsgpc_status gsgpc_group_allreduce_stats(gsgpc_group* group, gsgpc_stats** stats);
/* save_stats / load_stats (io.hpp:82-97, io.cpp:192-262), "GSGPSST1" layout. */
gsgpc_status gsgpc_stats_save(gsgpc_ctx* ctx, gsgpc_stats* stats, const char* path);
gsgpc_status gsgpc_stats_load(gsgpc_ctx* ctx, const char* path, gsgpc_stats** out);

/* ---------------------------------------------------------------- K_G operator */
/* ToeplitzOperator(Grid, KernelSpec) (grid.hpp:58-90) for the SE-ARD kernel
 * (kernels.hpp:11-47: noise_std, lengthscales[dim], outputscale). */
gsgpc_status gsgpc_kg_create(gsgpc_ctx* ctx, const gsgpc_grid* grid, const double* lengthscales,
                             double outputscale, double noise_std, gsgpc_kg** out);
/* The same with the K_G route chosen per dimension: dimensions with >= fft_min_nodes nodes
 * apply T_k by the reference's circulant embedding + FFT (grid.cpp:94-151, 193-235: zero-pad
 * to next_fast_fft_size(2 n_k − 1), r2c, spectrum product, c2r, 1/e scaling — per factor of
 * the separable kernel), the others by tensor-core Toeplitz mode products.  fft_min_nodes <= 0:
 * the default, 2041 (the mode products hold up to 2040 nodes per dimension). */
gsgpc_status gsgpc_kg_create_ex(gsgpc_ctx* ctx, const gsgpc_grid* grid, const double* lengthscales,
                                double outputscale, double noise_std, int64_t fft_min_nodes, gsgpc_kg** out);
/* next_fast_fft_size (grid.cpp:73-82): the smallest 5-smooth integer >= x (1 for x < 1). */
int64_t gsgpc_next_fast_fft_size(int64_t x);
void gsgpc_kg_destroy(gsgpc_kg* kg);
/* ToeplitzOperator::apply (grid.hpp:82-83, grid.cpp:193-235): out = K_G v. */
gsgpc_status gsgpc_kg_apply(gsgpc_ctx* ctx, gsgpc_kg* kg, const double* v, double* out);
gsgpc_status gsgpc_kg_info(const gsgpc_kg* kg, int64_t* m, double* noise_variance);

/* ---------------------------------------------------------------- solvers */
typedef struct {
  int32_t iterations;
  int32_t converged;
  double residual_sq;
  double loop_seconds; /* device time of the iteration loop (CUDA events) */
} gsgpc_solve_info;

/* factorized_cg_grid_rhs (solvers.hpp:127-151, solvers.cpp:271-336).  GridRhsTolerance:
 * eps_abs >= 0 wins, else rel_tol.  Traces (optional, host or device): residual_trace
 * maxiter+1, alphas maxiter, betas maxiter. */
gsgpc_status gsgpc_factorized_cg_grid_rhs(gsgpc_ctx* ctx, gsgpc_kg* kg, gsgpc_stats* stats,
                                          const double* rhat0, double sigma, double eps_abs,
                                          double rel_tol, int maxiter, double* xhat_d,
                                          gsgpc_solve_info* info, double* residual_trace,
                                          double* alphas, double* betas);
/* posterior_mean_gsgp (gp.hpp:119-122, gp.cpp:326-352): mean_coeffs = K_G(x̂_d + W^T y/σ²).
 * Returns NONCONVERGENCE (info filled) when maxiter is hit. */
gsgpc_status gsgpc_posterior_mean_gsgp(gsgpc_ctx* ctx, gsgpc_stats* stats, gsgpc_kg* kg,
                                       double sigma, double tol, int maxiter,
                                       double* mean_coeffs, gsgpc_solve_info* info);
/* PosteriorModel::predict_mean (gp.hpp:112-113, gp.cpp:309-324). */
gsgpc_status gsgpc_predict_mean(gsgpc_ctx* ctx, const gsgpc_grid* grid, int scheme,
                                const double* mean_coeffs, const gsgpc_points* pts, int64_t n,
                                double* out);

/* factorized_lanczos_fused (solvers.hpp:178-183, solvers.cpp:464-538) for P start vectors at
 * once (probe-batched EFLA).  kgwt_z0 / wt_z0 are P × m, z0_sq P.  Outputs per probe:
 * alpha P × k, beta P × k (first order-1 used), order P. */
gsgpc_status gsgpc_factorized_lanczos_fused(gsgpc_ctx* ctx, gsgpc_kg* kg, gsgpc_stats* stats,
                                            int probes, const double* kgwt_z0,
                                            const double* wt_z0, const double* z0_sq,
                                            double sigma_sq, int k, double* alpha,
                                            double* beta, int32_t* order);

typedef struct {
  double solve_tol;   /* LoglikOptions::solve_tol (gp.hpp:75) */
  int32_t probes;     /* LoglikOptions::probes */
  int32_t max_depth;  /* SlqOptions::max_depth (gp.hpp:25-29) */
  double quad_tol;    /* SlqOptions::quad_tol */
  uint64_t seed;      /* LoglikOptions::seed */
  int32_t maxiter;    /* LoglikOptions::maxiter */
  int32_t route;      /* LoglikOptions::route (gp.hpp:55-60): GSGPC_ROUTE_* */
  int64_t dense_cap;  /* LoglikOptions::dense_cap (default 2048) */
  /* SLQ probe shard [probe_begin, probe_end) of the `probes` probes (0, 0: all).  Ranks that
   * split the probes add their slq_sum / slq_count (gsgpc_loglik_result) to combine. */
  int32_t probe_begin, probe_end;
} gsgpc_loglik_options;

/* LogdetRoute (gp.hpp:55-60) */
enum {
  GSGPC_ROUTE_AUTO = 0,           /* SkiOperator when probe images exist, else by conditioning */
  GSGPC_ROUTE_SYMMETRIC_GRID = 1, /* SLQ(K WᵀW K + σ²K) − SLQ(K), m-dimensional probes */
  GSGPC_ROUTE_SKI_OPERATOR = 2,   /* factorized SLQ over the precompute's probe images */
  GSGPC_ROUTE_DENSE = 3           /* LU of K WᵀW + σ²I, m ≤ dense_cap */
};

typedef struct {
  double loglik, logdet_term, quad_term, const_term; /* LoglikResult (gp.hpp:62-72) */
  int32_t probes_used;
  int32_t solver_iterations;
  int32_t max_depth_used;
  int32_t logdet_route;  /* the route taken (GSGPC_ROUTE_*, never AUTO) */
  /* probe-shard combine: logdet_term = slq_sum / slq_count + logdet_shift over the whole probe
   * set (SkiOperator: shift −(n − m) log σ²; SymmetricGrid: sum of SLQ(sym) − SLQ(K) per probe;
   * Dense: slq_count = 0, logdet_term exact) */
  double slq_sum;
  int32_t slq_count;
  double logdet_shift;
} gsgpc_loglik_result;

/* log_likelihood_gsgp (gp.hpp:86-90, gp.cpp:158-240).  Routes as the reference:
 * SkiOperator = slq_logdet_ski_factorized (gp.cpp:85-111) over the probe images W^T v_p
 * accumulated during the precompute (gsgpc_stats_enable_probes: the reference's
 * rademacher_probe streams, gp.cpp:16-25) — the analogue of passing W; SymmetricGrid =
 * slq_logdet (gp.cpp:67-83) of K WᵀW K + σ²K minus that of K with m-dimensional probes and
 * quad_tol 0; Dense = dense_logdet_grid_system (gp.cpp:116-140); Auto picks SkiOperator
 * when the statistics carry probe images, else Dense if
 * estimate_grid_kernel_condition (gp.cpp:142-154) > 1e8 and m ≤ dense_cap, else
 * SymmetricGrid. */
gsgpc_status gsgpc_log_likelihood_gsgp(gsgpc_ctx* ctx, gsgpc_stats* stats, gsgpc_kg* kg,
                                       double sigma, const gsgpc_loglik_options* opts,
                                       gsgpc_loglik_result* out);

/* ---- posterior covariance (gp.cpp:381-528) */
/* posterior_cov_exact (gp.cpp:381-427) for the model (stats, kg, sigma): one grid-rhs EFCG per
 * test point (rel_tol = tol; the right-hand sides run batched, 32 per pass, one stencil read
 * per iteration for all of them), cov(i,j) = w_iᵀK_G w_j − (K_G w_i)·x̂_j, symmetrised
 * (cov, ns × ns row-major).  max_asymmetry / total_iterations may be NULL.  Errors:
 * OUT_OF_GRID "interp_weights: ..." (row = test point), BREAKDOWN, NONCONVERGENCE
 * "posterior_cov_exact: solver hit maxiter". */
gsgpc_status gsgpc_posterior_cov_exact(gsgpc_ctx* ctx, gsgpc_stats* stats, gsgpc_kg* kg, double sigma,
                                       const gsgpc_points* pts, int64_t ns, double tol, int maxiter, double* cov,
                                       double* max_asymmetry, int32_t* total_iterations);
/* posterior_cov_lowrank (gp.cpp:429-475): EFLA of depth `rank` from ĝ = WᵀW1/‖WᵀW1‖ with
 * the basis kept; the handle holds R = K_G(WᵀW Q̂ + d·WᵀWĝ/√(ĝᵀWᵀWĝ)) (device, rank × m),
 * the tridiagonal T and its own copy of the K_G generators (LowRankCov, gp.hpp:148-167). */
typedef struct gsgpc_lowrank gsgpc_lowrank;
gsgpc_status gsgpc_posterior_cov_lowrank(gsgpc_ctx* ctx, gsgpc_stats* stats, gsgpc_kg* kg, double sigma,
                                         int64_t rank, gsgpc_lowrank** out);
void gsgpc_lowrank_destroy(gsgpc_lowrank* lr);
/* LowRankCov::rank() — the Lanczos order reached (≤ rank). */
gsgpc_status gsgpc_lowrank_rank(const gsgpc_lowrank* lr, int64_t* rank);
/* LowRankCov::cov_matrix (gp.cpp:500-525), ns × ns row-major, symmetrised. */
gsgpc_status gsgpc_lowrank_cov_matrix(gsgpc_ctx* ctx, gsgpc_lowrank* lr, const gsgpc_points* pts, int64_t ns,
                                      double* cov);
/* LowRankCov::query (gp.cpp:486-498): cov between two points (d doubles each). */
gsgpc_status gsgpc_lowrank_query(gsgpc_ctx* ctx, gsgpc_lowrank* lr, const double* x, const double* x2, double* out);

#ifdef __cplusplus
}
#endif
#endif /* GSGPC_H */
