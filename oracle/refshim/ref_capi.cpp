// ref_capi.cpp — TEST INFRASTRUCTURE.  The orc_* C entry points of oracle/gsgp_oracle.h
// implemented by CALLING THE REFERENCE'S OWN CODE (the unmodified sources under
// /root/reference/proj, compiled where they lie against the stand-in headers of this
// directory — oracle/refshim/README.md), so that the same Python binding and the same tests
// can run against either the restatement (libgsgp_oracle.so) or the reference
// (oracle/_ref/libgsgp_ref.so).  Built by `make -C oracle ref`; never part of the product.
//
// gp.cpp is included as a source file (not copied) because rademacher_probe,
// quadrature_logdet, estimate_grid_kernel_condition and dense_logdet_grid_system live in its
// anonymous namespace; the other reference sources are separate translation units.
#include "gp.cpp"  // NOLINT  (found through -I /root/reference/proj/src)

#include <cstring>
#include <memory>
#include <string>
#include <thread>

#include "../gsgp_oracle.h"

namespace {

using gsgp::Grid;
using gsgp::GridDim;
using gsgp::InterpScheme;
using Eigen::Index;
using Eigen::MatrixXd;
using Eigen::VectorXd;

thread_local std::string g_err;
thread_local int64_t g_err_row = 0;

template <class F>
int guard(F&& f) {
  try {
    f();
    return ORC_OK;
  } catch (const gsgp::SolverBreakdown& e) {
    g_err = e.what();
    return ORC_BREAKDOWN;
  } catch (const gsgp::SolverNonConvergence& e) {
    g_err = e.what();
    return ORC_NONCONVERGENCE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    // the reference reports out-of-grid points as std::invalid_argument with these texts
    // (interp.cpp:52-54, 120-124); "stream row N" is added by sufficient_stats (interp.cpp:256-259)
    const bool oog = g_err.find("point outside grid") != std::string::npos ||
                     g_err.find("stencil leaves the grid") != std::string::npos;
    const auto p = g_err.find("stream row ");
    if (p != std::string::npos) g_err_row = std::strtoll(g_err.c_str() + p + 11, nullptr, 10);
    return oog ? ORC_OUT_OF_GRID : ORC_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ORC_RUNTIME_ERROR;
  }
}

Grid make_grid(int d, const double* gmin, const double* gmax, const int64_t* gsize) {
  std::vector<GridDim> dims(d);
  for (int k = 0; k < d; ++k) dims[k] = GridDim{gmin[k], gmax[k], static_cast<Index>(gsize[k])};
  return Grid(std::move(dims));
}

InterpScheme scheme_of(int s) { return s == 0 ? InterpScheme::Linear : InterpScheme::Cubic; }

VectorXd vec(const double* p, Index n) {
  VectorXd v(n);
  for (Index i = 0; i < n; ++i) v[i] = p[i];
  return v;
}

void put(double* dst, const VectorXd& v) {
  if (v.size() > 0) std::memcpy(dst, v.data(), sizeof(double) * static_cast<std::size_t>(v.size()));
}

// rows of an array as the reference's RowStream (interp.hpp:150-155)
template <class T>
class ArrayStream : public gsgp::RowStream {
 public:
  ArrayStream(int d, const T* x, const T* y, int64_t n) : d_(d), x_(x), y_(y), n_(n) {}
  int dim() const override { return d_; }
  bool next(VectorXd& x, double& y) override {
    if (i_ >= n_) return false;
    for (int k = 0; k < d_; ++k) x[k] = static_cast<double>(x_[i_ * d_ + k]);
    y = static_cast<double>(y_[i_]);
    ++i_;
    return true;
  }

 private:
  int d_;
  const T *x_, *y_;
  int64_t n_, i_ = 0;
};

// nthreads == 1: the reference's sufficient_stats (one pass in stream order).  nthreads > 1:
// one SufficientStatsAccumulator per row shard, combined with the reference's merge()
// (interp.cpp:202-210) in shard order, then finalize().
template <class T>
gsgp::SufficientStats run_stats(const Grid& grid, InterpScheme scheme, const T* x, const T* y, int64_t n,
                                int nthreads) {
  const int d = grid.dim();
  if (nthreads < 1) nthreads = 1;
  if (n < 1024 * nthreads) nthreads = 1;
  if (nthreads == 1) {
    ArrayStream<T> st(d, x, y, n);
    return gsgp::sufficient_stats(grid, scheme, st);
  }
  std::vector<std::unique_ptr<gsgp::SufficientStatsAccumulator>> accs(nthreads);
  std::vector<int64_t> bad_row(nthreads, -1);
  std::vector<std::string> bad_msg(nthreads);
  auto work = [&](int t) {
    const int64_t lo = n * t / nthreads, hi = n * (t + 1) / nthreads;
    accs[t] = std::make_unique<gsgp::SufficientStatsAccumulator>(grid, scheme);
    VectorXd xv(d);
    for (int64_t i = lo; i < hi; ++i) {
      for (int k = 0; k < d; ++k) xv[k] = static_cast<double>(x[i * d + k]);
      try {
        accs[t]->add(xv, static_cast<double>(y[i]));
      } catch (const std::invalid_argument& e) {
        bad_row[t] = i + 1;
        bad_msg[t] = e.what();
        return;
      }
    }
  };
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t) th.emplace_back(work, t);
  for (auto& h : th) h.join();
  for (int t = 0; t < nthreads; ++t) {
    if (bad_row[t] >= 0) {
      throw std::invalid_argument("sufficient_stats: stream row " + std::to_string(bad_row[t]) + ": " + bad_msg[t]);
    }
  }
  for (int t = 1; t < nthreads; ++t) accs[0]->merge(*accs[t]);
  return accs[0]->finalize();
}

// non-owning shared_ptr views for the PosteriorModel entry points
template <class T>
std::shared_ptr<const T> borrow(const T* p) {
  return std::shared_ptr<const T>(std::shared_ptr<const T>(), p);
}

using LoglikFn5 = gsgp::LoglikResult (*)(const gsgp::SufficientStats&, const gsgp::ToeplitzOperator&, double,
                                         const gsgp::LoglikOptions&, const gsgp::InterpMatrix*);

}  // namespace

struct orc_stats {
  gsgp::SufficientStats s;
};
struct orc_kg {
  std::unique_ptr<gsgp::ToeplitzOperator> t;
  gsgp::KernelSpec spec;
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int64_t orc_last_error_row(void) { return g_err_row; }
/* identifies this library as the reference build (the restatement does not export it) */
const char* orc_ref_build(void) { return "reference sources: kernels.cpp grid.cpp interp.cpp solvers.cpp gp.cpp"; }

int orc_fit_grid_to_data(int d, const double* lo, const double* hi, const int64_t* sizes, int scheme, double* out_min,
                         double* out_max) {
  return guard([&] {
    std::vector<Index> sz(sizes, sizes + d);
    const Grid g = gsgp::fit_grid_to_data(vec(lo, d), vec(hi, d), sz, scheme_of(scheme));
    for (int k = 0; k < d; ++k) {
      out_min[k] = g.min(k);
      out_max[k] = g.max(k);
    }
  });
}

int orc_interp_weights(int d, const double* gmin, const double* gmax, const int64_t* gsize, int scheme,
                       const double* x, int64_t* idx, double* w, int* nnz) {
  return guard([&] {
    const Grid g = make_grid(d, gmin, gmax, gsize);
    const gsgp::WeightVector wv = gsgp::interp_weights(g, vec(x, d), scheme_of(scheme));
    for (std::size_t i = 0; i < wv.indices.size(); ++i) {
      idx[i] = wv.indices[i];
      w[i] = wv.values[i];
    }
    *nnz = static_cast<int>(wv.indices.size());
  });
}

int orc_sufficient_stats(int d, const double* gmin, const double* gmax, const int64_t* gsize, int scheme,
                         const double* x, const double* y, int64_t n, int nthreads, orc_stats** out) {
  g_err_row = 0;
  return guard([&] {
    const Grid g = make_grid(d, gmin, gmax, gsize);
    *out = new orc_stats{run_stats(g, scheme_of(scheme), x, y, n, nthreads)};
  });
}

int orc_sufficient_stats_f32(int d, const double* gmin, const double* gmax, const int64_t* gsize, int scheme,
                             const float* x, const float* y, int64_t n, int nthreads, orc_stats** out) {
  g_err_row = 0;
  return guard([&] {
    const Grid g = make_grid(d, gmin, gmax, gsize);
    *out = new orc_stats{run_stats(g, scheme_of(scheme), x, y, n, nthreads)};
  });
}

void orc_stats_destroy(orc_stats* s) { delete s; }

void orc_stats_info(const orc_stats* s, int64_t* m, int64_t* n, int64_t* nnz, double* yty) {
  *m = s->s.grid_size();
  *n = s->s.n();
  *nnz = s->s.wtw().nonZeros();
  *yty = s->s.yty();
}

void orc_stats_export(const orc_stats* s, int64_t* row_ptr, int64_t* col, double* val, double* wty) {
  const auto& a = s->s.wtw();
  const Index m = a.rows(), nnz = a.nonZeros();
  if (row_ptr)
    for (Index i = 0; i <= m; ++i) row_ptr[i] = a.outerIndexPtr()[i];
  if (col)
    for (Index k = 0; k < nnz; ++k) col[k] = a.innerIndexPtr()[k];
  if (val)
    for (Index k = 0; k < nnz; ++k) val[k] = a.valuePtr()[k];
  if (wty) put(wty, s->s.wty());
}

int orc_stats_from_csr(int64_t m, int64_t nnz, const int64_t* row_ptr, const int64_t* col, const double* val,
                       const double* wty, double yty, int64_t n, orc_stats** out) {
  return guard([&] {
    std::vector<Eigen::Triplet<double>> trips;
    trips.reserve(static_cast<std::size_t>(nnz));
    for (int64_t i = 0; i < m; ++i)
      for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
        trips.emplace_back(static_cast<int>(i), static_cast<int>(col[k]), val[k]);
    Eigen::SparseMatrix<double, Eigen::RowMajor> a(m, m);
    a.setFromTriplets(trips.begin(), trips.end());
    *out = new orc_stats{gsgp::SufficientStats(std::move(a), vec(wty, m), yty, n)};
  });
}

int orc_stats_apply_wtw(const orc_stats* s, const double* v, double* out) {
  return guard([&] { put(out, s->s.apply_wtw(vec(v, s->s.grid_size()))); });
}

int64_t orc_stats_max_row_nnz(const orc_stats* s) { return s->s.max_row_nnz(); }

int orc_kg_create(int d, const double* gmin, const double* gmax, const int64_t* gsize, const double* lengthscales,
                  double outputscale, double noise_std, orc_kg** out) {
  return guard([&] {
    const Grid g = make_grid(d, gmin, gmax, gsize);
    gsgp::KernelSpec spec(gsgp::Hyperparams(noise_std, vec(lengthscales, d), outputscale));
    auto t = std::make_unique<gsgp::ToeplitzOperator>(gsgp::build_toeplitz_operator(g, spec));
    *out = new orc_kg{std::move(t), spec};
  });
}

void orc_kg_destroy(orc_kg* k) { delete k; }

int64_t orc_kg_dim(const orc_kg* k) { return k->t->dim(); }

void orc_kg_embed_shape(const orc_kg* k, int64_t* shape) {  // grid.cpp:97-103
  const Grid& g = k->t->grid();
  for (int i = 0; i < g.dim(); ++i) shape[i] = gsgp::next_fast_fft_size(2 * g.size(i) - 1);
}

int orc_kg_apply(const orc_kg* k, const double* v, double* out) {
  return guard([&] { put(out, k->t->apply(vec(v, k->t->dim()))); });
}

int orc_kernel_generator(const orc_kg* k, double* out) {
  return guard([&] { put(out, gsgp::kernel_generator_tensor(k->spec, k->t->grid())); });
}

int orc_kg_dense(const orc_kg* k, double* out, int64_t max_points) {
  return guard([&] {
    const MatrixXd K = gsgp::kg_dense(k->t->grid(), k->spec, max_points);
    const Index m = K.rows();
    for (Index i = 0; i < m; ++i)
      for (Index j = 0; j < m; ++j) out[i * m + j] = K(i, j);
  });
}

int64_t orc_next_fast_fft_size(int64_t x) { return gsgp::next_fast_fft_size(x); }

/* restatement-only diagnostics: no counterpart in the reference */
void orc_kg_set_direct(orc_kg*, int) {}
void orc_set_threads(int) {}
int orc_get_threads(void) { return 1; }

int orc_factorized_cg_grid_rhs(const orc_kg* kg, const orc_stats* st, const double* rhat0, double sigma,
                               double eps_abs, double rel_tol, int maxiter, double* xhat_d, int* iterations,
                               int* converged, double* residual_sq, double* residual_trace, double* alphas,
                               double* betas, double* loop_seconds) {
  return guard([&] {
    gsgp::GridRhsTolerance tol;
    tol.eps_abs = eps_abs;
    tol.rel_tol = rel_tol;
    const gsgp::GridSolveResult r =
        gsgp::factorized_cg_grid_rhs(*kg->t, st->s, vec(rhat0, kg->t->dim()), sigma, tol, maxiter);
    put(xhat_d, r.xhat_d);
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
    *residual_sq = r.residual_sq;
    if (residual_trace)
      std::memcpy(residual_trace, r.residual_trace.data(), sizeof(double) * r.residual_trace.size());
    if (alphas) std::memcpy(alphas, r.alphas.data(), sizeof(double) * r.alphas.size());
    if (betas) std::memcpy(betas, r.betas.data(), sizeof(double) * r.betas.size());
    if (loop_seconds) *loop_seconds = r.loop_seconds;
  });
}

int orc_posterior_mean_gsgp(const orc_kg* kg, const orc_stats* st, double sigma, double tol, int maxiter,
                            double* mean_coeffs, int* iterations, double* residual_sq) {
  return guard([&] {
    const gsgp::PosteriorModel model = gsgp::posterior_mean_gsgp(borrow(&st->s), borrow(kg->t.get()), kg->spec,
                                                                 InterpScheme::Cubic, sigma, tol, maxiter);
    put(mean_coeffs, model.mean_coeffs);
    if (iterations) *iterations = model.solve_iterations;
    if (residual_sq) *residual_sq = model.solve_residual_sq;
  });
}

int orc_predict_mean(int d, const double* gmin, const double* gmax, const int64_t* gsize, int scheme,
                     const double* mean_coeffs, const double* pts, int64_t npts, double* out) {
  return guard([&] {
    // PosteriorModel::predict_mean (gp.cpp:309-324) takes its grid from the model's K_G: any
    // valid kernel on the same grid serves
    const Grid g = make_grid(d, gmin, gmax, gsize);
    gsgp::KernelSpec spec(gsgp::Hyperparams(1.0, VectorXd::Ones(d), 1.0));
    const gsgp::ToeplitzOperator kg = gsgp::build_toeplitz_operator(g, spec);
    gsgp::PosteriorModel model;
    model.scheme = scheme_of(scheme);
    model.mean_coeffs = vec(mean_coeffs, g.num_points());
    model.kg = borrow(&kg);
    MatrixXd P(npts, d);
    for (int64_t p = 0; p < npts; ++p)
      for (int k = 0; k < d; ++k) P(p, k) = pts[p * d + k];
    put(out, model.predict_mean(P));
  });
}

void orc_rademacher_probe(int64_t n, uint64_t seed, uint64_t probe_index, double* out) {
  put(out, gsgp::rademacher_probe(n, seed, probe_index));
}

void orc_rademacher_bits(int64_t n, uint64_t seed, int probes, uint64_t* words, int) {
  std::memset(words, 0, sizeof(uint64_t) * static_cast<std::size_t>(n));
  for (int p = 0; p < probes; ++p) {
    const VectorXd v = gsgp::rademacher_probe(n, seed, static_cast<uint64_t>(p));
    for (int64_t i = 0; i < n; ++i)
      if (v[i] > 0.0) words[i] |= (1ull << p);
  }
}

int orc_wt_apply(int d, const double* gmin, const double* gmax, const int64_t* gsize, int scheme, const double* x,
                 int64_t n, const double* u, double* out) {
  return guard([&] {
    const Grid g = make_grid(d, gmin, gmax, gsize);
    MatrixXd P(n, d);
    for (int64_t p = 0; p < n; ++p)
      for (int k = 0; k < d; ++k) P(p, k) = x[p * d + k];
    const gsgp::InterpMatrix w = gsgp::build_interp_matrix(g, P, scheme_of(scheme));
    put(out, w.apply_transpose(vec(u, n)));
  });
}

int orc_factorized_lanczos_fused(const orc_kg* kg, const orc_stats* st, const double* kgwt_z0, const double* wt_z0,
                                 double z0_sq, double sigma_sq, int k, double* alpha, double* beta, double* dvec,
                                 double* basis, int* order) {
  return guard([&] {
    const Index m = kg->t->dim();
    gsgp::FactorizedBasis b;
    b.kgwt_z0 = vec(kgwt_z0, m);
    b.wt_z0 = vec(wt_z0, m);
    b.z0_sq = z0_sq;
    b.sigma_sq = sigma_sq;
    const gsgp::TridiagonalFactor t = gsgp::factorized_lanczos_fused(*kg->t, st->s, b, k);
    *order = t.order();
    put(alpha, t.alpha);
    put(beta, t.beta);
    if (dvec) put(dvec, t.d);
    if (basis)
      for (Index j = 0; j < t.basis.cols() && j < t.order(); ++j) put(basis + j * m, t.basis.col(j));
  });
}

int orc_quadrature_logdet(const double* alpha, const double* beta, int k, double probe_sq, double quad_tol,
                          double* value, int* depth) {
  return guard([&] {
    gsgp::TridiagonalFactor t;
    t.alpha = vec(alpha, k);
    t.beta = vec(beta, k > 1 ? k - 1 : 0);
    gsgp::SlqOptions o;
    o.quad_tol = quad_tol;
    const auto q = gsgp::quadrature_logdet(t, probe_sq, o);
    *value = q.value;
    *depth = q.depth;
  });
}

/* the stand-in's own tridiagonal solver — not reference code; kept so the binding loads */
int orc_tridiag_eig(int k, const double* alpha, const double* beta, double* evals, double* first_row) {
  return guard([&] {
    Eigen::SelfAdjointEigenSolver<MatrixXd> es;
    es.computeFromTridiagonal(vec(alpha, k), vec(beta, k > 1 ? k - 1 : 0));
    put(evals, es.eigenvalues());
    for (int l = 0; l < k; ++l) first_row[l] = es.eigenvectors()(0, l);
  });
}

int orc_slq_logdet_ski_factorized(const orc_kg* kg, const orc_stats* st, int d, const double* gmin,
                                  const double* gmax, const int64_t* gsize, int scheme, const double* x, int64_t n,
                                  double sigma, int num_probes, int max_depth, double quad_tol, uint64_t seed,
                                  double* logdet, int* max_depth_used) {
  return guard([&] {
    const Grid g = make_grid(d, gmin, gmax, gsize);
    MatrixXd P(n, d);
    for (int64_t p = 0; p < n; ++p)
      for (int k = 0; k < d; ++k) P(p, k) = x[p * d + k];
    const gsgp::InterpMatrix w = gsgp::build_interp_matrix(g, P, scheme_of(scheme));
    gsgp::SlqOptions o;
    o.max_depth = max_depth;
    o.quad_tol = quad_tol;
    const gsgp::SlqResult r = gsgp::slq_logdet_ski_factorized(*kg->t, w, st->s, sigma, num_probes, o, seed);
    *logdet = r.logdet;
    *max_depth_used = r.max_depth_used;
  });
}

int orc_log_likelihood_gsgp(const orc_stats* st, const orc_kg* kg, double sigma, double solve_tol, int probes,
                            int max_depth, double quad_tol, uint64_t seed, int route, int64_t dense_cap, int maxiter,
                            int d, const double* gmin, const double* gmax, const int64_t* gsize, int scheme,
                            const double* x, int64_t n, double* out, int* iout) {
  return guard([&] {
    gsgp::LoglikOptions o;
    o.solve_tol = solve_tol;
    o.probes = probes;
    o.slq.max_depth = max_depth;
    o.slq.quad_tol = quad_tol;
    o.seed = seed;
    o.route = route == 1   ? gsgp::LogdetRoute::SymmetricGrid
              : route == 2 ? gsgp::LogdetRoute::SkiOperator
              : route == 3 ? gsgp::LogdetRoute::Dense
                           : gsgp::LogdetRoute::Auto;
    o.dense_cap = dense_cap;
    o.maxiter = maxiter;
    std::unique_ptr<gsgp::InterpMatrix> w;
    if (x != nullptr) {
      const Grid g = make_grid(d, gmin, gmax, gsize);
      MatrixXd P(n, d);
      for (int64_t p = 0; p < n; ++p)
        for (int k = 0; k < d; ++k) P(p, k) = x[p * d + k];
      w = std::make_unique<gsgp::InterpMatrix>(gsgp::build_interp_matrix(g, P, scheme_of(scheme)));
    }
    // the 5-parameter definition (gp.cpp:158-240); the header declares a 6-parameter overload
    const LoglikFn5 fn = &gsgp::log_likelihood_gsgp;
    const gsgp::LoglikResult r = fn(st->s, *kg->t, sigma, o, w.get());
    out[0] = r.loglik;
    out[1] = r.logdet_term;
    out[2] = r.quad_term;
    out[3] = r.const_term;
    iout[0] = r.probes_used;
    iout[1] = r.solver_iterations;
    iout[2] = r.logdet_route == "symmetric-grid-slq" ? 1 : r.logdet_route == "ski-operator-slq" ? 2 : 3;
  });
}

int orc_posterior_cov_exact(const orc_kg* kg, const orc_stats* st, int scheme, double sigma, const double* pts,
                            int64_t ns, double tol, int maxiter, double* cov, double* max_asym, int* total_iters) {
  return guard([&] {
    const int d = kg->t->grid().dim();
    gsgp::PosteriorModel model;
    model.spec = kg->spec;
    model.scheme = scheme_of(scheme);
    model.sigma = sigma;
    model.kg = borrow(kg->t.get());
    model.stats = borrow(&st->s);
    MatrixXd P(ns, d);
    for (int64_t p = 0; p < ns; ++p)
      for (int k = 0; k < d; ++k) P(p, k) = pts[p * d + k];
    const gsgp::CovResult c = gsgp::posterior_cov_exact(model, P, tol, maxiter);
    for (int64_t i = 0; i < ns; ++i)
      for (int64_t j = 0; j < ns; ++j) cov[i * ns + j] = c.cov(i, j);
    *max_asym = c.max_asymmetry;
    *total_iters = c.total_iterations;
  });
}

int orc_posterior_cov_lowrank(const orc_kg* kg, const orc_stats* st, int scheme, double sigma, int64_t rank,
                              const double* pts, int64_t ns, double* cov, const double* qx, const double* qx2,
                              double* qout, int* rank_used) {
  return guard([&] {
    const int d = kg->t->grid().dim();
    gsgp::PosteriorModel model;
    model.spec = kg->spec;
    model.scheme = scheme_of(scheme);
    model.sigma = sigma;
    model.kg = borrow(kg->t.get());
    model.stats = borrow(&st->s);
    const gsgp::LowRankCov lr = gsgp::posterior_cov_lowrank(model, rank);
    *rank_used = static_cast<int>(lr.rank());
    if (ns > 0) {
      MatrixXd P(ns, d);
      for (int64_t p = 0; p < ns; ++p)
        for (int k = 0; k < d; ++k) P(p, k) = pts[p * d + k];
      const MatrixXd c = lr.cov_matrix(P);
      for (int64_t i = 0; i < ns; ++i)
        for (int64_t j = 0; j < ns; ++j) cov[i * ns + j] = c(i, j);
    }
    if (qx && qx2 && qout) *qout = lr.query(vec(qx, d), vec(qx2, d));
  });
}

}  // extern "C"
