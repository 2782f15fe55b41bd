/*
 * gsgp_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference hot path (arXiv 2101.11751 C++ reference at
 * /root/reference/proj, namespace gsgp).  Only tests/, __graft_entry__.smoke() and
 * bench.py (cpu_baseline leg and --impl reference) may load this library, and only as
 * the checker / CPU baseline — never as the product path.
 *
 * Parity status: the reference's own build cannot run in this image (Eigen3, FFTW3 and
 * nlohmann-json absent) and its own tests are empty stubs.  This restatement is
 * pinned against (1) the reference's OWN SOURCES compiled where they lie against self-written
 * stand-ins for those headers (oracle/refshim, oracle/_ref/libgsgp_ref.so exporting these same
 * entry points; tests/test_ref_pin.py) and (2) the SPEC.md known-answer examples and
 * independent numpy fixtures (tests/golden/).  Unpinned: the bit pattern of real Eigen's /
 * FFTW's internal reductions.
 *
 * Every entry point cites the reference function it restates (file:line under
 * /root/reference/proj).  Errors are returned as codes (see ORC_*), never thrown across
 * the C boundary; orc_last_error() holds the reference's message text.
 */
#ifndef GSGP_ORACLE_H
#define GSGP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_INVALID_ARGUMENT = 1,
  ORC_OUT_OF_GRID = 2,    /* "point outside grid" / "stencil leaves the grid" */
  ORC_BREAKDOWN = 3,      /* SolverBreakdown */
  ORC_NONCONVERGENCE = 4, /* SolverNonConvergence */
  ORC_RUNTIME_ERROR = 7,
};

typedef struct orc_stats orc_stats;
typedef struct orc_kg orc_kg;

const char* orc_last_error(void);
int64_t orc_last_error_row(void);

/* interp.cpp:286-306 */
int orc_fit_grid_to_data(int d, const double* lo, const double* hi, const int64_t* sizes,
                         int scheme, double* out_min, double* out_max);

/* interp.cpp:79-134 — weights of one point; idx/w need room for 4^d entries. */
int orc_interp_weights(int d, const double* gmin, const double* gmax, const int64_t* gsize,
                       int scheme, const double* x, int64_t* idx, double* w, int* nnz);

/* interp.cpp:244-263 (single pass, stream order) with SufficientStatsAccumulator
 * (interp.cpp:179-221).  x is n×d row-major fp64, y is n fp64.  nthreads>1 shards the
 * rows and combines shards with merge() (interp.cpp:202-210). */
int orc_sufficient_stats(int d, const double* gmin, const double* gmax, const int64_t* gsize,
                         int scheme, const double* x, const double* y, int64_t n,
                         int nthreads, orc_stats** out);
/* Same from fp32 inputs widened to fp64 (configs 2–4 store fp32). */
int orc_sufficient_stats_f32(int d, const double* gmin, const double* gmax,
                             const int64_t* gsize, int scheme, const float* x,
                             const float* y, int64_t n, int nthreads, orc_stats** out);
void orc_stats_destroy(orc_stats* s);
/* m, n, nnz(WtW), yty */
void orc_stats_info(const orc_stats* s, int64_t* m, int64_t* n, int64_t* nnz, double* yty);
/* RowMajor CSR export (row_ptr m+1, col nnz, val nnz) and W^T y. */
void orc_stats_export(const orc_stats* s, int64_t* row_ptr, int64_t* col, double* val,
                      double* wty);
/* Build stats from CSR arrays (used by the stats-file loader tests). */
int orc_stats_from_csr(int64_t m, int64_t nnz, const int64_t* row_ptr, const int64_t* col,
                       const double* val, const double* wty, double yty, int64_t n,
                       orc_stats** out);
/* SufficientStats::apply_wtw (interp.cpp:227-233). */
int orc_stats_apply_wtw(const orc_stats* s, const double* v, double* out);
int64_t orc_stats_max_row_nnz(const orc_stats* s);

/* ToeplitzOperator (grid.cpp:94-151) with the SE kernel (kernels.cpp:43-55). */
int orc_kg_create(int d, const double* gmin, const double* gmax, const int64_t* gsize,
                  const double* lengthscales, double outputscale, double noise_std,
                  orc_kg** out);
void orc_kg_destroy(orc_kg* k);
int64_t orc_kg_dim(const orc_kg* k);
/* embed shape e_k = next_fast_fft_size(2 m_k - 1) (grid.cpp:73-82) */
void orc_kg_embed_shape(const orc_kg* k, int64_t* shape);
/* ToeplitzOperator::apply (grid.cpp:193-235). */
int orc_kg_apply(const orc_kg* k, const double* v, double* out);
/* kernel_generator_tensor (grid.cpp:42-52) and kg_dense (grid.cpp:54-71). */
int orc_kernel_generator(const orc_kg* k, double* out);
int orc_kg_dense(const orc_kg* k, double* out, int64_t max_points);
int64_t orc_next_fast_fft_size(int64_t x);
/* Sensitivity study only: K_G v by direct separable Toeplitz sums instead of the circulant
 * FFT (same operator, different rounding).  Not the reference algorithm. */
void orc_kg_set_direct(orc_kg* k, int direct);
/* Host threads for independent rows / FFT lines / SLQ probes (results do not depend on it). */
void orc_set_threads(int n);
int orc_get_threads(void);

/* factorized_cg_grid_rhs (solvers.cpp:271-336).  Traces need room for maxiter+1. */
int orc_factorized_cg_grid_rhs(const orc_kg* kg, const orc_stats* st, const double* rhat0,
                               double sigma, double eps_abs, double rel_tol, int maxiter,
                               double* xhat_d, int* iterations, int* converged,
                               double* residual_sq, double* residual_trace, double* alphas,
                               double* betas, double* loop_seconds);

/* posterior_mean_gsgp (gp.cpp:326-352): mean_coeffs = K_G(x̂_d + W^T y/σ²). */
int orc_posterior_mean_gsgp(const orc_kg* kg, const orc_stats* st, double sigma, double tol,
                            int maxiter, double* mean_coeffs, int* iterations,
                            double* residual_sq);

/* PosteriorModel::predict_mean (gp.cpp:309-324). pts is npts×d row-major. */
int orc_predict_mean(int d, const double* gmin, const double* gmax, const int64_t* gsize,
                     int scheme, const double* mean_coeffs, const double* pts, int64_t npts,
                     double* out);

/* rademacher_probe (gp.cpp:16-25). */
void orc_rademacher_probe(int64_t n, uint64_t seed, uint64_t probe_index, double* out);
/* Bit-packed probes: word[i] bit p = (p-th probe, i-th draw is +1). P <= 64. */
void orc_rademacher_bits(int64_t n, uint64_t seed, int probes, uint64_t* words, int nthreads);

/* InterpMatrix::apply_transpose restated as a stream: W^T u over the n points. */
int orc_wt_apply(int d, const double* gmin, const double* gmax, const int64_t* gsize,
                 int scheme, const double* x, int64_t n, const double* u, double* out);

/* factorized_lanczos_fused (solvers.cpp:464-538).  alpha k, beta k-1, d k, basis m×k
 * (column-major, may be NULL); *order receives the completed order. */
int orc_factorized_lanczos_fused(const orc_kg* kg, const orc_stats* st, const double* kgwt_z0,
                                 const double* wt_z0, double z0_sq, double sigma_sq, int k,
                                 double* alpha, double* beta, double* dvec, double* basis,
                                 int* order);

/* quadrature_logdet (gp.cpp:34-63). */
int orc_quadrature_logdet(const double* alpha, const double* beta, int k, double probe_sq,
                          double quad_tol, double* value, int* depth);

/* Symmetric tridiagonal eigen-decomposition: eigenvalues ascending + first eigenvector row. */
int orc_tridiag_eig(int k, const double* alpha, const double* beta, double* evals,
                    double* first_row);

/* slq_logdet_ski_factorized (gp.cpp:85-111) with W^T v streamed over the points. */
int orc_slq_logdet_ski_factorized(const orc_kg* kg, const orc_stats* st, int d,
                                  const double* gmin, const double* gmax, const int64_t* gsize,
                                  int scheme, const double* x, int64_t n, double sigma,
                                  int num_probes, int max_depth, double quad_tol, uint64_t seed,
                                  double* logdet, int* max_depth_used);

/* log_likelihood_gsgp (gp.cpp:158-240, the 5-parameter definition).  route: 0 Auto,
 * 1 SymmetricGrid, 2 SkiOperator, 3 Dense.  x may be NULL (no W). out[0..3] = loglik,
 * logdet_term, quad_term, const_term; iout[0..2] = probes_used, solver_iterations,
 * route taken. */
int orc_log_likelihood_gsgp(const orc_stats* st, const orc_kg* kg, double sigma,
                            double solve_tol, int probes, int max_depth, double quad_tol,
                            uint64_t seed, int route, int64_t dense_cap, int maxiter, int d,
                            const double* gmin, const double* gmax, const int64_t* gsize,
                            int scheme, const double* x, int64_t n, double* out, int* iout);

/* posterior_cov_exact (gp.cpp:381-427): cov ns×ns symmetrised, max asymmetry, Σ iterations. */
int orc_posterior_cov_exact(const orc_kg* kg, const orc_stats* st, int scheme, double sigma, const double* pts,
                            int64_t ns, double tol, int maxiter, double* cov, double* max_asym, int* total_iters);
/* posterior_cov_lowrank (gp.cpp:429-475) + LowRankCov::cov_matrix / query (gp.cpp:486-525). */
int orc_posterior_cov_lowrank(const orc_kg* kg, const orc_stats* st, int scheme, double sigma, int64_t rank,
                              const double* pts, int64_t ns, double* cov, const double* qx, const double* qx2,
                              double* qout, int* rank_used);

#ifdef __cplusplus
}
#endif
#endif
