// gsgp_b200.hpp — C++17 host API mirroring the reference's gsgp:: hot path
// (/root/reference/proj/include/gsgp/*.hpp) on top of the C ABI (gsgpc.h, libgsgpc.so).
//
// Same names, argument meaning and error behaviour as the reference:
//   Grid / GridDim / fit_grid_to_data ............ grid.hpp:15-44, interp.hpp:168-172
//   InterpScheme / interp_weights ................ interp.hpp:15-41
//   SufficientStatsAccumulator / SufficientStats /
//   sufficient_stats / RowStream ................. interp.hpp:87-160
//   Hyperparams / KernelSpec ..................... kernels.hpp:11-32
//   ToeplitzOperator ............................. grid.hpp:58-90
//   GridRhsTolerance / GridSolveResult /
//   factorized_cg_grid_rhs ....................... solvers.hpp:118-151
//   PosteriorModel / posterior_mean_gsgp ......... gp.hpp:101-122
//   SlqOptions / LoglikOptions / LoglikResult /
//   log_likelihood_gsgp .......................... gp.hpp:25-90
//   save_stats / load_stats ...................... io.hpp:82-97
// Eigen::VectorXd / MatrixXd become std::vector<double> (row-major point matrices); the
// exceptions are the reference's: std::invalid_argument, SolverBreakdown,
// SolverNonConvergence, std::runtime_error.  All compute runs on the GPU (no CPU path).
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gsgpc.h"

namespace gsgp_b200 {

class SolverBreakdown : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

class SolverNonConvergence : public std::runtime_error {
 public:
  SolverNonConvergence(const std::string& what, double r, int it)
      : std::runtime_error(what), residual_sq(r), iterations(it) {}
  double residual_sq;
  int iterations;
};

// ---------------------------------------------------------------- context
class Context {
 public:
  explicit Context(int device = 0) {
    gsgpc_ctx* c = nullptr;
    if (gsgpc_ctx_create(device, &c) != GSGPC_OK) throw std::runtime_error("gsgpc: no CUDA device " + std::to_string(device));
    h_.reset(c, gsgpc_ctx_destroy);
  }
  gsgpc_ctx* get() const { return h_.get(); }
  void check(gsgpc_status st, double residual_sq = NAN, int iterations = 0) const {
    if (st == GSGPC_OK) return;
    const std::string msg = gsgpc_last_error(h_.get());
    switch (st) {
      case GSGPC_INVALID_ARGUMENT:
      case GSGPC_OUT_OF_GRID:
        throw std::invalid_argument(msg);
      case GSGPC_BREAKDOWN:
        throw SolverBreakdown(msg);
      case GSGPC_NONCONVERGENCE:
        throw SolverNonConvergence(msg, residual_sq, iterations);
      default:
        throw std::runtime_error(msg);
    }
  }
  int64_t last_error_row() const { return gsgpc_last_error_row(h_.get()); }
  static Context& default_context() {
    static Context ctx(0);
    return ctx;
  }
  // A context owned by someone else (a DeviceGroup), kept alive through `owner`.
  Context(std::shared_ptr<void> owner, gsgpc_ctx* borrowed) : h_(std::move(owner), borrowed) {}

 private:
  std::shared_ptr<gsgpc_ctx> h_;
};

// ---------------------------------------------------------------- grid (grid.hpp:15-44)
struct GridDim {
  double min = 0.0;
  double max = 1.0;
  int64_t size = 2;
};

class Grid {
 public:
  Grid() = default;
  explicit Grid(std::vector<GridDim> dims) : dims_(std::move(dims)) {
    if (dims_.empty()) throw std::invalid_argument("Grid: need at least one dimension");
    total_ = 1;
    for (const auto& d : dims_) {
      if (d.size < 2) throw std::invalid_argument("Grid: size must be >= 2 per dimension");
      if (!(d.max > d.min)) throw std::invalid_argument("Grid: max must exceed min");
      spacings_.push_back((d.max - d.min) / static_cast<double>(d.size - 1));
      total_ *= d.size;
    }
  }
  int dim() const { return static_cast<int>(dims_.size()); }
  int64_t size(int d) const { return dims_[d].size; }
  double min(int d) const { return dims_[d].min; }
  double max(int d) const { return dims_[d].max; }
  double spacing(int d) const { return spacings_[d]; }
  int64_t num_points() const { return total_; }
  const std::vector<GridDim>& dims() const { return dims_; }
  int64_t flat_index(const std::vector<int64_t>& multi) const {
    int64_t f = 0;
    for (int d = 0; d < dim(); ++d) f = f * dims_[d].size + multi[d];
    return f;
  }
  std::vector<double> point(int64_t flat) const {
    std::vector<double> x(dim());
    for (int d = dim() - 1; d >= 0; --d) {
      const int64_t i = flat % dims_[d].size;
      flat /= dims_[d].size;
      x[d] = dims_[d].min + static_cast<double>(i) * spacings_[d];
    }
    return x;
  }
  gsgpc_grid c() const {
    if (dim() > GSGPC_MAX_DIM) throw std::runtime_error("gsgp_b200: grids of dimension > 3 are not supported");
    gsgpc_grid g{};
    g.dim = dim();
    for (int k = 0; k < dim(); ++k) {
      g.min[k] = dims_[k].min;
      g.max[k] = dims_[k].max;
      g.size[k] = dims_[k].size;
    }
    return g;
  }

 private:
  std::vector<GridDim> dims_;
  std::vector<double> spacings_;
  int64_t total_ = 0;
};

enum class InterpScheme { Linear = GSGPC_LINEAR, Cubic = GSGPC_CUBIC };

inline int stencil_radius(InterpScheme s) { return s == InterpScheme::Linear ? 1 : 2; }

// interp.cpp:286-306
inline Grid fit_grid_to_data(const std::vector<double>& lo, const std::vector<double>& hi,
                             const std::vector<int64_t>& sizes, InterpScheme scheme) {
  if (lo.size() != hi.size() || lo.size() != sizes.size()) {
    throw std::invalid_argument("fit_grid_to_data: dimension mismatch");
  }
  const int r = stencil_radius(scheme);
  std::vector<GridDim> dims(sizes.size());
  for (size_t k = 0; k < sizes.size(); ++k) {
    const int64_t m = sizes[k];
    if (m < 2 * r + 2) {
      throw std::invalid_argument("fit_grid_to_data: need at least " + std::to_string(2 * r + 2) +
                                  " points per dimension");
    }
    if (!(hi[k] > lo[k])) throw std::invalid_argument("fit_grid_to_data: empty data range");
    const double s = (hi[k] - lo[k]) / static_cast<double>(m - 1 - 2 * r);
    dims[k] = GridDim{lo[k] - r * s, hi[k] + r * s, m};
  }
  return Grid(std::move(dims));
}

// ---------------------------------------------------------------- kernels.hpp:11-32
struct Hyperparams {
  double noise_std = 1.0;
  std::vector<double> lengthscales;
  double outputscale = 1.0;
  Hyperparams() = default;
  Hyperparams(double noise, std::vector<double> ls, double os)
      : noise_std(noise), lengthscales(std::move(ls)), outputscale(os) {
    if (!(noise_std > 0.0)) throw std::invalid_argument("Hyperparams: noise_std must be positive");
    if (lengthscales.empty()) throw std::invalid_argument("Hyperparams: need at least one lengthscale");
    for (double l : lengthscales) {
      if (!(l > 0.0)) throw std::invalid_argument("Hyperparams: lengthscales must be positive");
    }
    if (!(outputscale > 0.0)) throw std::invalid_argument("Hyperparams: outputscale must be positive");
  }
  int dim() const { return static_cast<int>(lengthscales.size()); }
  double noise_variance() const { return noise_std * noise_std; }
};

struct KernelSpec {
  Hyperparams hyper;
  KernelSpec() = default;
  explicit KernelSpec(Hyperparams h) : hyper(std::move(h)) {}
};

// ---------------------------------------------------------------- interp weights
struct WeightVector {
  std::vector<int64_t> indices;
  std::vector<double> values;
  InterpScheme scheme = InterpScheme::Cubic;
  int64_t nnz() const { return static_cast<int64_t>(indices.size()); }
};

inline WeightVector interp_weights(const Grid& grid, const std::vector<double>& x, InterpScheme scheme,
                                   Context& ctx = Context::default_context()) {
  if (static_cast<int>(x.size()) != grid.dim()) throw std::invalid_argument("interp_weights: dimension mismatch");
  const gsgpc_grid g = grid.c();
  gsgpc_points p{};
  p.dtype = GSGPC_F64;
  p.x = x.data();
  p.x_row_stride = grid.dim();
  for (int k = 0; k < grid.dim(); ++k) p.x_col_offset[k] = k;
  p.y = x.data();
  int width = 1;
  for (int k = 0; k < grid.dim(); ++k) width *= 2 * stencil_radius(scheme);
  std::vector<int64_t> idx(width);
  std::vector<double> w(width);
  int32_t nnz = 0, status = 0;
  ctx.check(gsgpc_interp_weights(ctx.get(), &g, static_cast<int>(scheme), &p, 1, idx.data(), w.data(), &nnz, &status));
  if (status == 1) throw std::invalid_argument("interp_weights: point outside grid");
  if (status == 2) {
    throw std::invalid_argument(
        "interp_weights: stencil leaves the grid (point too close to the boundary for the requested scheme)");
  }
  WeightVector out;
  out.scheme = scheme;
  out.indices.assign(idx.begin(), idx.begin() + nnz);
  out.values.assign(w.begin(), w.begin() + nnz);
  return out;
}

// ---------------------------------------------------------------- sufficient statistics
class SufficientStats {
 public:
  SufficientStats() = default;
  SufficientStats(std::shared_ptr<gsgpc_stats> h, Grid grid, InterpScheme scheme, Context ctx)
      : h_(std::move(h)), grid_(std::move(grid)), scheme_(scheme), ctx_(std::move(ctx)) {}

  int64_t grid_size() const { return grid_.num_points(); }
  const Grid& grid() const { return grid_; }
  InterpScheme scheme() const { return scheme_; }
  gsgpc_stats* handle() const { return h_.get(); }
  const Context& context() const { return ctx_; }

  std::vector<double> wty() const {
    std::vector<double> out(grid_size());
    ctx_.check(gsgpc_stats_copy_wty(ctx_.get(), h_.get(), out.data()));
    return out;
  }
  double yty() const {
    double v = 0.0;
    ctx_.check(gsgpc_stats_info(ctx_.get(), h_.get(), nullptr, nullptr, &v, nullptr, nullptr));
    return v;
  }
  int64_t n() const {
    int64_t v = 0;
    ctx_.check(gsgpc_stats_info(ctx_.get(), h_.get(), nullptr, &v, nullptr, nullptr, nullptr));
    return v;
  }
  // SufficientStats::wtw() (interp.hpp:129) as RowMajor CSR arrays.
  struct Csr {
    std::vector<int64_t> row_ptr, col;
    std::vector<double> val;
  };
  Csr wtw() const {
    int64_t nnz = 0, mx = 0;
    ctx_.check(gsgpc_stats_csr_nnz(ctx_.get(), h_.get(), &nnz, &mx));
    Csr c;
    c.row_ptr.resize(grid_size() + 1);
    c.col.resize(nnz);
    c.val.resize(nnz);
    ctx_.check(gsgpc_stats_export_csr(ctx_.get(), h_.get(), c.row_ptr.data(), c.col.data(), c.val.data()));
    return c;
  }
  std::vector<double> apply_wtw(const std::vector<double>& v) const {
    if (static_cast<int64_t>(v.size()) != grid_size()) {
      throw std::invalid_argument("SufficientStats::apply_wtw: length mismatch");
    }
    std::vector<double> out(grid_size());
    ctx_.check(gsgpc_stats_apply_wtw(ctx_.get(), h_.get(), v.data(), out.data()));
    ++wtw_count_;
    return out;
  }
  int64_t max_row_nnz() const {
    int64_t nnz = 0, mx = 0;
    ctx_.check(gsgpc_stats_csr_nnz(ctx_.get(), h_.get(), &nnz, &mx));
    return mx;
  }
  int64_t matvec_count() const { return wtw_count_; }

 private:
  std::shared_ptr<gsgpc_stats> h_;
  Grid grid_;
  InterpScheme scheme_ = InterpScheme::Cubic;
  Context ctx_{Context::default_context()};
  mutable int64_t wtw_count_ = 0;
};

// ---------------------------------------------------------------- several GPUs, one process
// gsgpc_group_* (SURVEY §8(b) gsgpc_ctx_create(device_ids[], ngpu)): sufficient_stats sharded
// by rows over the devices and combined with one all-reduce — merge() semantics
// (interp.cpp:202-210) — so every device holds the full statistics.
class DeviceGroup {
 public:
  explicit DeviceGroup(const std::vector<int>& devices) {
    gsgpc_group* g = nullptr;
    if (devices.empty() || gsgpc_group_create(devices.data(), static_cast<int>(devices.size()), &g) != GSGPC_OK)
      throw std::runtime_error("gsgpc: cannot create a device group");
    h_.reset(g, gsgpc_group_destroy);
  }
  int size() const {
    int n = 0;
    gsgpc_group_info(h_.get(), &n, nullptr);
    return n;
  }
  bool uses_nccl() const {
    int u = 0;
    gsgpc_group_info(h_.get(), nullptr, &u);
    return u != 0;
  }
  Context context(int rank) const { return Context(h_, gsgpc_group_ctx(h_.get(), rank)); }
  // x: n × d row-major coordinates, y: n responses.
  std::vector<SufficientStats> sufficient_stats(const Grid& grid, InterpScheme scheme, const std::vector<double>& x,
                                                const std::vector<double>& y, int probes = 0,
                                                uint64_t seed = 0) const {
    const int d = grid.dim();
    if (static_cast<int64_t>(x.size()) != static_cast<int64_t>(y.size()) * d)
      throw std::invalid_argument("sufficient_stats: stream/grid dimension mismatch");
    gsgpc_points p{};
    p.dtype = GSGPC_F64;
    p.x = x.data();
    p.x_row_stride = d;
    for (int k = 0; k < d; ++k) p.x_col_offset[k] = k;
    p.y = y.data();
    p.y_stride = 1;
    const gsgpc_grid g = grid.c();
    std::vector<gsgpc_stats*> out(size(), nullptr);
    const gsgpc_status st =
        gsgpc_group_sufficient_stats(h_.get(), &g, scheme == InterpScheme::Linear ? GSGPC_LINEAR : GSGPC_CUBIC, &p,
                                     static_cast<int64_t>(y.size()), probes, seed, out.data());
    if (st == GSGPC_INVALID_ARGUMENT || st == GSGPC_OUT_OF_GRID)
      throw std::invalid_argument(gsgpc_group_last_error(h_.get()));
    if (st != GSGPC_OK) throw std::runtime_error(gsgpc_group_last_error(h_.get()));
    std::vector<SufficientStats> res;
    for (int r = 0; r < static_cast<int>(out.size()); ++r)
      res.emplace_back(std::shared_ptr<gsgpc_stats>(out[r], gsgpc_stats_destroy), grid, scheme, context(r));
    return res;
  }

 private:
  std::shared_ptr<gsgpc_group> h_;
};

// Row-at-a-time data source (interp.hpp:150-155).  sufficient_stats() drains it in
// batches and ships each batch to the GPU.
class RowStream {
 public:
  virtual ~RowStream() = default;
  virtual int dim() const = 0;
  virtual bool next(std::vector<double>& x, double& y) = 0;
};

// GSGPDAT1 dataset file (io.hpp:31-45): 8-byte magic "GSGPDAT1", u64 n, u64 d, then n rows
// of (d+1) little-endian doubles.  The constructor validates the header (io.cpp:103-113);
// sufficient_stats() hands the whole file to the library (gsgpc_stats_add_file: reader
// thread + pinned double buffers overlapped with the precompute); next() also works.
class BinaryRowStream : public RowStream {
 public:
  explicit BinaryRowStream(const std::string& path) : path_(path), file_(path, std::ios::binary) {
    if (!file_) throw std::invalid_argument("cannot open binary dataset: " + path);
    char magic[8];
    if (!file_.read(magic, 8) || std::memcmp(magic, "GSGPDAT1", 8) != 0) {
      throw std::invalid_argument("bad magic in binary dataset: " + path);
    }
    uint64_t v = 0;
    if (!file_.read(reinterpret_cast<char*>(&v), 8)) throw std::invalid_argument("truncated file while reading row count");
    n_ = static_cast<int64_t>(v);
    if (!file_.read(reinterpret_cast<char*>(&v), 8)) throw std::invalid_argument("truncated file while reading dimension");
    dim_ = static_cast<int>(v);
    if (v < 1 || v > 64) throw std::invalid_argument("binary dataset: bad dimension");
  }
  int dim() const override { return dim_; }
  int64_t rows() const { return n_; }
  const std::string& path() const { return path_; }
  int64_t rows_read() const { return read_; }
  bool next(std::vector<double>& x, double& y) override {
    if (read_ >= n_) return false;
    x.resize(dim_);
    for (int k = 0; k < dim_; ++k) {
      if (!file_.read(reinterpret_cast<char*>(&x[k]), 8)) throw std::invalid_argument("truncated file while reading coordinate");
    }
    if (!file_.read(reinterpret_cast<char*>(&y), 8)) throw std::invalid_argument("truncated file while reading response");
    ++read_;
    return true;
  }

 private:
  std::string path_;
  std::ifstream file_;
  int dim_ = 0;
  int64_t n_ = 0;
  int64_t read_ = 0;
};

class SufficientStatsAccumulator {
 public:
  SufficientStatsAccumulator(Grid grid, InterpScheme scheme, Context ctx = Context::default_context())
      : grid_(std::move(grid)), scheme_(scheme), ctx_(std::move(ctx)) {
    const gsgpc_grid g = grid_.c();
    gsgpc_stats* s = nullptr;
    ctx_.check(gsgpc_stats_create(ctx_.get(), &g, static_cast<int>(scheme), &s));
    h_.reset(s, gsgpc_stats_destroy);
  }
  // add(x, y) of interp.cpp:188-200, for one row ...
  void add(const std::vector<double>& x, double y) { add_rows(x.data(), &y, 1); }
  // ... or a batch of n rows (x row-major n × d, y n), host or device memory.
  void add_rows(const double* x, const double* y, int64_t n) {
    gsgpc_points p{};
    p.dtype = GSGPC_F64;
    p.x = x;
    p.x_row_stride = grid_.dim();
    for (int k = 0; k < grid_.dim(); ++k) p.x_col_offset[k] = k;
    p.y = y;
    p.y_stride = 1;
    ctx_.check(gsgpc_stats_add(ctx_.get(), h_.get(), &p, n, nullptr, 0));
    rows_ += n;
  }
  void add_points(const gsgpc_points& p, int64_t n) {
    ctx_.check(gsgpc_stats_add(ctx_.get(), h_.get(), &p, n, nullptr, 0));
    rows_ += n;
  }
  // every row of a GSGPDAT1 file; returns the rows added
  int64_t add_file(const std::string& path) {
    int64_t rows = 0;
    ctx_.check(gsgpc_stats_add_file(ctx_.get(), h_.get(), path.c_str(), &rows));
    rows_ += rows;
    return rows;
  }
  void enable_probes(int probes, uint64_t seed) {
    ctx_.check(gsgpc_stats_enable_probes(ctx_.get(), h_.get(), probes, seed));
  }
  void merge(const SufficientStatsAccumulator& other) {
    ctx_.check(gsgpc_stats_merge(ctx_.get(), h_.get(), other.h_.get()));
    rows_ += other.rows_;
  }
  SufficientStats finalize() const {
    ctx_.check(gsgpc_stats_finalize(ctx_.get(), h_.get()));
    return SufficientStats(h_, grid_, scheme_, ctx_);
  }
  int64_t rows_seen() const { return rows_; }

 private:
  Grid grid_;
  InterpScheme scheme_;
  Context ctx_;
  std::shared_ptr<gsgpc_stats> h_;
  int64_t rows_ = 0;
};

// interp.cpp:244-263 — one pass over the stream; errors carry the 1-based stream row.
inline SufficientStats sufficient_stats(const Grid& grid, InterpScheme scheme, RowStream& stream,
                                        Context ctx = Context::default_context()) {
  if (stream.dim() != grid.dim()) {
    throw std::invalid_argument("sufficient_stats: stream/grid dimension mismatch");
  }
  SufficientStatsAccumulator acc(grid, scheme, ctx);
  if (auto* bin = dynamic_cast<BinaryRowStream*>(&stream)) {
    if (bin->rows_read() == 0) {  // whole file through the library's overlapped reader
      acc.add_file(bin->path());
      return acc.finalize();
    }
  }
  const int d = grid.dim();
  const int64_t batch = int64_t{1} << 20;
  std::vector<double> xs, ys, x(d);
  double y = 0.0;
  xs.reserve(batch * d);
  ys.reserve(batch);
  auto flush = [&] {
    if (!ys.empty()) acc.add_rows(xs.data(), ys.data(), static_cast<int64_t>(ys.size()));
    xs.clear();
    ys.clear();
  };
  while (stream.next(x, y)) {
    xs.insert(xs.end(), x.begin(), x.end());
    ys.push_back(y);
    if (static_cast<int64_t>(ys.size()) == batch) flush();
  }
  flush();
  return acc.finalize();
}

// ---------------------------------------------------------------- K_G (grid.hpp:58-90)
class ToeplitzOperator {
 public:
  ToeplitzOperator(const Grid& grid, const KernelSpec& spec, Context ctx = Context::default_context())
      : grid_(grid), ctx_(std::move(ctx)), sigma_sq_(spec.hyper.noise_variance()) {
    if (spec.hyper.dim() != grid.dim()) {
      throw std::invalid_argument("build_toeplitz_operator: kernel/grid dimension mismatch");
    }
    const gsgpc_grid g = grid.c();
    gsgpc_kg* k = nullptr;
    ctx_.check(gsgpc_kg_create(ctx_.get(), &g, spec.hyper.lengthscales.data(), spec.hyper.outputscale,
                               spec.hyper.noise_std, &k));
    h_.reset(k, gsgpc_kg_destroy);
  }
  int64_t dim() const { return grid_.num_points(); }
  double noise_variance() const { return sigma_sq_; }
  const Grid& grid() const { return grid_; }
  gsgpc_kg* handle() const { return h_.get(); }
  std::vector<double> apply(const std::vector<double>& v) const {
    if (static_cast<int64_t>(v.size()) != dim()) throw std::invalid_argument("ToeplitzOperator::apply: length mismatch");
    std::vector<double> out(dim());
    ctx_.check(gsgpc_kg_apply(ctx_.get(), h_.get(), v.data(), out.data()));
    ++count_;
    return out;
  }
  int64_t matvec_count() const { return count_; }

 private:
  Grid grid_;
  Context ctx_;
  double sigma_sq_;
  std::shared_ptr<gsgpc_kg> h_;
  mutable int64_t count_ = 0;
};

// ---------------------------------------------------------------- solvers.hpp:118-151
constexpr int kDefaultMaxIter = 1000;

struct GridRhsTolerance {
  double eps_abs = -1.0;
  double rel_tol = -1.0;
};

struct GridSolveResult {
  std::vector<double> xhat_d;
  int iterations = 0;
  bool converged = false;
  double residual_sq = 0.0;
  std::vector<double> residual_trace;
  std::vector<double> alphas;
  std::vector<double> betas;
  double loop_seconds = 0.0;
};

inline GridSolveResult factorized_cg_grid_rhs(const ToeplitzOperator& kg, const SufficientStats& stats,
                                              const std::vector<double>& rhat0, double sigma, GridRhsTolerance tol,
                                              int maxiter = kDefaultMaxIter) {
  if (static_cast<int64_t>(rhat0.size()) != kg.dim()) {
    throw std::invalid_argument("factorized_cg_grid_rhs: dimension mismatch");
  }
  GridSolveResult r;
  r.xhat_d.resize(kg.dim());
  std::vector<double> tr(maxiter + 1), al(maxiter + 1), be(maxiter + 1);
  gsgpc_solve_info info{};
  stats.context().check(gsgpc_factorized_cg_grid_rhs(stats.context().get(), kg.handle(), stats.handle(), rhat0.data(),
                                                     sigma, tol.eps_abs, tol.rel_tol, maxiter, r.xhat_d.data(), &info,
                                                     tr.data(), al.data(), be.data()));
  r.iterations = info.iterations;
  r.converged = info.converged != 0;
  r.residual_sq = info.residual_sq;
  r.loop_seconds = info.loop_seconds;
  r.residual_trace.assign(tr.begin(), tr.begin() + r.iterations + 1);
  r.alphas.assign(al.begin(), al.begin() + r.iterations);
  const int nb = r.converged ? std::max(0, r.iterations - 1) : r.iterations;
  r.betas.assign(be.begin(), be.begin() + nb);
  return r;
}

// ---------------------------------------------------------------- gp.hpp:101-122
struct PosteriorModel {
  KernelSpec spec;
  InterpScheme scheme = InterpScheme::Cubic;
  double sigma = 1.0;
  std::vector<double> mean_coeffs;
  std::shared_ptr<const ToeplitzOperator> kg;
  std::shared_ptr<const SufficientStats> stats;
  int solve_iterations = 0;
  double solve_residual_sq = 0.0;
  std::string fit_path;

  const Grid& grid() const { return kg->grid(); }
  // predict_mean for a batch of points (row-major npts × d), gp.cpp:309-324.
  std::vector<double> predict_mean(const std::vector<double>& points) const {
    const int d = grid().dim();
    const int64_t np = static_cast<int64_t>(points.size()) / d;
    const gsgpc_grid g = grid().c();
    gsgpc_points p{};
    p.dtype = GSGPC_F64;
    p.x = points.data();
    p.x_row_stride = d;
    for (int k = 0; k < d; ++k) p.x_col_offset[k] = k;
    p.y = points.data();
    std::vector<double> out(np);
    const Context& ctx = stats ? stats->context() : Context::default_context();
    ctx.check(gsgpc_predict_mean(ctx.get(), &g, static_cast<int>(scheme), mean_coeffs.data(), &p, np, out.data()));
    return out;
  }
  double predict_mean_point(const std::vector<double>& x) const { return predict_mean(x)[0]; }
};

inline PosteriorModel posterior_mean_gsgp(std::shared_ptr<const SufficientStats> stats,
                                          std::shared_ptr<const ToeplitzOperator> kg, KernelSpec spec,
                                          InterpScheme scheme, double sigma, double tol,
                                          int maxiter = kDefaultMaxIter) {
  if (!stats || !kg) throw std::invalid_argument("posterior_mean_gsgp: null inputs");
  PosteriorModel model;
  model.mean_coeffs.resize(kg->dim());
  gsgpc_solve_info info{};
  const gsgpc_status st = gsgpc_posterior_mean_gsgp(stats->context().get(), stats->handle(), kg->handle(), sigma, tol,
                                                    maxiter, model.mean_coeffs.data(), &info);
  stats->context().check(st, info.residual_sq, info.iterations);
  model.spec = std::move(spec);
  model.scheme = scheme;
  model.sigma = sigma;
  model.kg = std::move(kg);
  model.stats = std::move(stats);
  model.solve_iterations = info.iterations;
  model.solve_residual_sq = info.residual_sq;
  model.fit_path = "gsgp";
  return model;
}

// ---------------------------------------------------------------- gp.hpp:132-169 covariance
struct CovResult {
  std::vector<double> cov;  // ns × ns row-major
  double max_asymmetry = 0.0;
  int total_iterations = 0;
};

namespace detail {
inline gsgpc_points coords(const std::vector<double>& points, int d) {
  gsgpc_points p{};
  p.dtype = GSGPC_F64;
  p.x = points.data();
  p.x_row_stride = d;
  for (int k = 0; k < d; ++k) p.x_col_offset[k] = k;
  p.y = points.data();
  return p;
}
}  // namespace detail

// gp.cpp:381-427 (points row-major ns × d)
inline CovResult posterior_cov_exact(const PosteriorModel& model, const std::vector<double>& points, double tol,
                                     int maxiter = kDefaultMaxIter) {
  if (!model.stats) throw std::invalid_argument("posterior_cov_exact: the model carries no sufficient statistics");
  const int d = model.grid().dim();
  const int64_t ns = static_cast<int64_t>(points.size()) / d;
  const gsgpc_points p = detail::coords(points, d);
  CovResult r;
  r.cov.assign(static_cast<size_t>(ns * ns), 0.0);
  int32_t it = 0;
  const Context& ctx = model.stats->context();
  ctx.check(gsgpc_posterior_cov_exact(ctx.get(), model.stats->handle(), model.kg->handle(), model.sigma, &p, ns, tol,
                                      maxiter, r.cov.data(), &r.max_asymmetry, &it));
  r.total_iterations = it;
  return r;
}

class LowRankCov {
 public:
  int64_t rank() const {
    int64_t r = 0;
    if (h_) gsgpc_lowrank_rank(h_.get(), &r);
    return r;
  }
  double query(const std::vector<double>& x, const std::vector<double>& x2) const {
    double out = 0.0;
    ctx_.check(gsgpc_lowrank_query(ctx_.get(), h_.get(), x.data(), x2.data(), &out));
    return out;
  }
  std::vector<double> cov_matrix(const std::vector<double>& points) const {
    const int64_t ns = static_cast<int64_t>(points.size()) / d_;
    const gsgpc_points p = detail::coords(points, d_);
    std::vector<double> cov(static_cast<size_t>(ns * ns));
    ctx_.check(gsgpc_lowrank_cov_matrix(ctx_.get(), h_.get(), &p, ns, cov.data()));
    return cov;
  }

 private:
  friend LowRankCov posterior_cov_lowrank(const PosteriorModel&, int64_t);
  std::shared_ptr<gsgpc_lowrank> h_;
  Context ctx_{Context::default_context()};
  int d_ = 1;
};

// gp.cpp:429-475
inline LowRankCov posterior_cov_lowrank(const PosteriorModel& model, int64_t rank) {
  if (!model.stats) throw std::invalid_argument("posterior_cov_lowrank: the model carries no sufficient statistics");
  LowRankCov out;
  out.ctx_ = model.stats->context();
  out.d_ = model.grid().dim();
  gsgpc_lowrank* h = nullptr;
  out.ctx_.check(gsgpc_posterior_cov_lowrank(out.ctx_.get(), model.stats->handle(), model.kg->handle(), model.sigma,
                                             rank, &h));
  out.h_.reset(h, gsgpc_lowrank_destroy);
  return out;
}

// ---------------------------------------------------------------- gp.hpp:25-90
struct SlqOptions {
  int max_depth = 100;
  double quad_tol = 0.01;
};

enum class LogdetRoute { Auto = 0, SymmetricGrid = 1, SkiOperator = 2, Dense = 3 };  // gp.hpp:55-60

struct LoglikOptions {
  double solve_tol = 0.01;
  int probes = 30;
  SlqOptions slq;
  uint64_t seed = 0;
  LogdetRoute route = LogdetRoute::Auto;
  int64_t dense_cap = 2048;
  int maxiter = kDefaultMaxIter;
  int probe_begin = 0, probe_end = 0;  // SLQ probe shard; (0, 0) = all probes
};

struct LoglikResult {
  double loglik = 0.0, logdet_term = 0.0, quad_term = 0.0, const_term = 0.0;
  int probes_used = 0;
  int solver_iterations = 0;
  std::string logdet_route = "ski-operator-slq";
  double slq_sum = 0.0;  // probe-shard combine: logdet = Σ slq_sum / Σ slq_count + logdet_shift
  int slq_count = 0;
  double logdet_shift = 0.0;
};

// gp.cpp:158-240.  The SkiOperator route reads probe images accumulated in the precompute
// (SufficientStatsAccumulator::enable_probes(opts.probes, opts.seed) before adding rows);
// SymmetricGrid / Dense need only the statistics; Auto chooses as the reference does.
inline LoglikResult log_likelihood_gsgp(const SufficientStats& stats, const ToeplitzOperator& kg, double sigma,
                                        const LoglikOptions& opts) {
  gsgpc_loglik_options o{};
  o.solve_tol = opts.solve_tol;
  o.probes = opts.probes;
  o.max_depth = opts.slq.max_depth;
  o.quad_tol = opts.slq.quad_tol;
  o.seed = opts.seed;
  o.maxiter = opts.maxiter;
  o.route = static_cast<int32_t>(opts.route);
  o.dense_cap = opts.dense_cap;
  o.probe_begin = opts.probe_begin;
  o.probe_end = opts.probe_end;
  gsgpc_loglik_result r{};
  stats.context().check(gsgpc_log_likelihood_gsgp(stats.context().get(), stats.handle(), kg.handle(), sigma, &o, &r));
  LoglikResult out;
  out.loglik = r.loglik;
  out.logdet_term = r.logdet_term;
  out.quad_term = r.quad_term;
  out.const_term = r.const_term;
  out.probes_used = r.probes_used;
  out.solver_iterations = r.solver_iterations;
  out.logdet_route = r.logdet_route == 1 ? "symmetric-grid-slq" : r.logdet_route == 3 ? "dense" : "ski-operator-slq";
  out.slq_sum = r.slq_sum;
  out.slq_count = r.slq_count;
  out.logdet_shift = r.logdet_shift;
  return out;
}

// ---------------------------------------------------------------- io.hpp:82-97
inline void save_stats(const std::string& path, const SufficientStats& stats, const Grid& grid, InterpScheme) {
  if (grid.num_points() != stats.grid_size()) {
    throw std::invalid_argument("save_stats: grid does not match the statistics");
  }
  stats.context().check(gsgpc_stats_save(stats.context().get(), stats.handle(), path.c_str()));
}

struct StatsFile {
  Grid grid;
  InterpScheme scheme = InterpScheme::Cubic;
  SufficientStats stats;
};

inline StatsFile load_stats(const std::string& path, Context ctx = Context::default_context()) {
  gsgpc_stats* s = nullptr;
  ctx.check(gsgpc_stats_load(ctx.get(), path.c_str(), &s));
  std::shared_ptr<gsgpc_stats> h(s, gsgpc_stats_destroy);
  gsgpc_grid g{};
  int scheme = 1;
  gsgpc_stats_grid(s, &g, &scheme);
  std::vector<GridDim> dims;
  for (int k = 0; k < g.dim; ++k) dims.push_back(GridDim{g.min[k], g.max[k], g.size[k]});
  Grid grid(dims);
  const InterpScheme sch = scheme == 0 ? InterpScheme::Linear : InterpScheme::Cubic;
  return StatsFile{grid, sch, SufficientStats(h, grid, sch, ctx)};
}

}  // namespace gsgp_b200
