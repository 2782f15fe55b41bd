// gsgp_oracle.cpp — TEST INFRASTRUCTURE ONLY (see gsgp_oracle.h for the contract).
//
// CPU restatement of the reference hot path of the arXiv 2101.11751 C++ reference
// (/root/reference/proj).  Each function follows the cited reference lines: same
// control flow, same floating-point expression order, same error semantics.  Eigen and
// FFTW are absent from this image, so:
//   * Eigen vectors are std::vector<double>; dots and axpys are sequential loops (Eigen's
//     SIMD reductions sum in a different order — differences are O(1e-16) relative);
//   * the sparse W^T W is a RowMajor CSR built exactly like setFromTriplets (sorted rows,
//     sorted columns within a row, values = the accumulated hash-map sums);
//   * FFTW's r2c/c2r is replaced by a self-written mixed-radix (2/3/5) complex FFT over
//     the same circulant embedding (the embedding sizes are 5-smooth by construction).
// Build: oracle/Makefile (g++ -O3 -ffp-contract=off, no -march, like the reference's
// Release build, CMakeLists.txt:8-10, so no FMA contraction).
#include "gsgp_oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstring>
#include <exception>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <utility>
#include <vector>

namespace {

thread_local std::string g_err;
thread_local int64_t g_err_row = 0;

using Vec = std::vector<double>;
using cplx = std::complex<double>;

struct OutOfGrid : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct SolverBreakdown : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SolverNonConvergence : std::runtime_error {
  SolverNonConvergence(const std::string& w, double r, int it)
      : std::runtime_error(w), residual_sq(r), iterations(it) {}
  double residual_sq;
  int iterations;
};

constexpr double kLog2Pi = 1.8378770664093453;  // gp.cpp:12

// Host threads for the row/line-parallel loops below (orc_set_threads).  Only loops whose
// iterations are independent (CSR rows, FFT lines, SLQ probes) run in parallel, and every
// reduction keeps its sequential order, so results do not depend on the thread count.
int g_threads = 1;
thread_local bool g_in_par = false;

template <class F>
void par_for(int64_t n, F&& f, int64_t grain = 64) {  // f(lo, hi) over [0, n)
  const int64_t nt = std::min<int64_t>(g_in_par ? 1 : g_threads, n / std::max<int64_t>(grain, 1));
  if (nt <= 1) {
    if (n > 0) f(int64_t(0), n);
    return;
  }
  std::vector<std::thread> th;
  for (int64_t t = 0; t < nt; ++t) {
    th.emplace_back([&, t] {
      g_in_par = true;
      f(n * t / nt, n * (t + 1) / nt);
      g_in_par = false;
    });
  }
  for (auto& h : th) h.join();
}

// ---------------------------------------------------------------- grid.cpp:12-40
struct Grid {
  int d = 0;
  std::vector<double> mn, mx, sp;
  std::vector<int64_t> sz;
  int64_t m = 0;
  Grid() = default;
  Grid(int d_, const double* gmin, const double* gmax, const int64_t* gsize) : d(d_) {
    if (d < 1) throw std::invalid_argument("Grid: need at least one dimension");
    m = 1;
    for (int k = 0; k < d; ++k) {
      if (gsize[k] < 2) throw std::invalid_argument("Grid: size must be >= 2 per dimension");
      if (!(gmax[k] > gmin[k])) throw std::invalid_argument("Grid: max must exceed min");
      mn.push_back(gmin[k]);
      mx.push_back(gmax[k]);
      sz.push_back(gsize[k]);
      sp.push_back((gmax[k] - gmin[k]) / static_cast<double>(gsize[k] - 1));
      m *= gsize[k];
    }
  }
  Vec point(int64_t flat) const {  // grid.cpp:33-40
    Vec x(d);
    for (int k = d - 1; k >= 0; --k) {
      const int64_t i = flat % sz[k];
      flat /= sz[k];
      x[k] = mn[k] + static_cast<double>(i) * sp[k];
    }
    return x;
  }
};

// ---------------------------------------------------------------- interp.cpp:27-75
double cubic_weight(double t) {
  const double a = std::abs(t);
  if (a <= 1.0) return (1.5 * a - 2.5) * a * a + 1.0;
  if (a < 2.0) return ((-0.5 * a + 2.5) * a - 4.0) * a + 2.0;
  return 0.0;
}
double linear_weight(double t) {
  const double a = std::abs(t);
  return a <= 1.0 ? 1.0 - a : 0.0;
}
struct Stencil1d {
  int64_t start;
  double w[4];
  int count;
};
constexpr double kSnapTol = 1e-9;

Stencil1d stencil_1d(double x, double gmin, double spacing, int64_t size, int scheme) {
  double u = (x - gmin) / spacing;
  const double r = std::round(u);
  if (std::abs(u - r) < kSnapTol) u = r;
  if (u < 0.0 || u > static_cast<double>(size - 1)) {
    throw OutOfGrid("interp_weights: point outside grid");
  }
  int64_t i0 = static_cast<int64_t>(std::floor(u));
  if (i0 > size - 2) i0 = size - 2;
  const double t = u - static_cast<double>(i0);
  Stencil1d s{};
  if (scheme == 0) {  // Linear
    s.start = i0;
    s.w[0] = linear_weight(t);
    s.w[1] = linear_weight(1.0 - t);
    s.count = 2;
  } else {
    s.start = i0 - 1;
    s.w[0] = cubic_weight(t + 1.0);
    s.w[1] = cubic_weight(t);
    s.w[2] = cubic_weight(1.0 - t);
    s.w[3] = cubic_weight(2.0 - t);
    s.count = 4;
  }
  return s;
}

struct WeightVector {
  std::vector<int64_t> indices;
  std::vector<double> values;
};

// interp.cpp:79-134
WeightVector interp_weights(const Grid& grid, const double* x, int scheme) {
  const int d = grid.d;
  std::vector<Stencil1d> per_dim(d);
  for (int k = 0; k < d; ++k) {
    per_dim[k] = stencil_1d(x[k], grid.mn[k], grid.sp[k], grid.sz[k], scheme);
  }
  WeightVector out;
  const int width = per_dim[0].count;
  std::vector<int> offs(d, 0);
  int64_t combos = 1;
  for (int k = 0; k < d; ++k) combos *= width;
  out.indices.reserve(combos);
  out.values.reserve(combos);
  for (int64_t c = 0; c < combos; ++c) {
    double w = 1.0;
    int64_t flat = 0;
    bool in_range = true;
    for (int k = 0; k < d; ++k) {
      const Stencil1d& s = per_dim[k];
      const double wk = s.w[offs[k]];
      if (wk == 0.0) {
        w = 0.0;
        break;
      }
      const int64_t j = s.start + offs[k];
      if (j < 0 || j >= grid.sz[k]) {
        in_range = false;
        break;
      }
      w *= wk;
      flat = flat * grid.sz[k] + j;
    }
    if (w != 0.0) {
      if (!in_range) {
        throw OutOfGrid(
            "interp_weights: stencil leaves the grid (point too close to the boundary "
            "for the requested scheme)");
      }
      out.indices.push_back(flat);
      out.values.push_back(w);
    }
    for (int k = d - 1; k >= 0; --k) {
      if (++offs[k] < width) break;
      offs[k] = 0;
    }
  }
  return out;
}

// ---------------------------------------------------------------- interp.cpp:179-233
struct Stats {
  int64_t m = 0;
  std::vector<int64_t> row_ptr, col;
  Vec val;
  Vec wty;
  double yty = 0.0;
  int64_t n = 0;

  Vec apply_wtw(const Vec& v) const {  // Eigen RowMajor sparse * dense: per-row sequential
    Vec out(m, 0.0);
    par_for(m, [&](int64_t lo, int64_t hi) {
      for (int64_t i = lo; i < hi; ++i) {
        double tmp = 0.0;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) tmp += val[k] * v[col[k]];
        out[i] = tmp;
      }
    });
    return out;
  }
};

struct Accumulator {
  Grid grid;
  int scheme;
  int64_t m;
  std::unordered_map<int64_t, double> wtw;
  Vec wty;
  double yty = 0.0;
  int64_t n = 0;

  Accumulator(const Grid& g, int s) : grid(g), scheme(s), m(g.m), wty(g.m, 0.0) {
    const int r = s == 0 ? 1 : 2;
    const double per_row = std::pow(4.0 * r - 1.0, grid.d);
    wtw.reserve(static_cast<std::size_t>(std::min(per_row * static_cast<double>(m), 1e7)));
  }
  void add(const double* x, double y) {  // interp.cpp:188-200
    const WeightVector w = interp_weights(grid, x, scheme);
    const int64_t k = static_cast<int64_t>(w.indices.size());
    for (int64_t a = 0; a < k; ++a) {
      const double wa = w.values[a];
      wty[w.indices[a]] += y * wa;
      for (int64_t b = 0; b < k; ++b) {
        wtw[w.indices[a] * m + w.indices[b]] += wa * w.values[b];
      }
    }
    yty += y * y;
    ++n;
  }
  void merge(const Accumulator& o) {  // interp.cpp:202-210
    if (o.m != m || o.scheme != scheme) {
      throw std::invalid_argument("SufficientStatsAccumulator::merge: mismatched shards");
    }
    for (const auto& kv : o.wtw) wtw[kv.first] += kv.second;
    for (int64_t i = 0; i < m; ++i) wty[i] += o.wty[i];
    yty += o.yty;
    n += o.n;
  }
  Stats finalize() const {  // interp.cpp:212-221 (setFromTriplets on unique keys)
    std::vector<std::pair<int64_t, double>> trips(wtw.begin(), wtw.end());
    std::sort(trips.begin(), trips.end(),
              [](const auto& a, const auto& b) { return a.first < b.first; });
    Stats s;
    s.m = m;
    s.row_ptr.assign(m + 1, 0);
    s.col.resize(trips.size());
    s.val.resize(trips.size());
    for (std::size_t i = 0; i < trips.size(); ++i) {
      const int64_t r = trips[i].first / m;
      s.col[i] = trips[i].first % m;
      s.val[i] = trips[i].second;
      s.row_ptr[r + 1]++;
    }
    for (int64_t i = 0; i < m; ++i) s.row_ptr[i + 1] += s.row_ptr[i];
    s.wty = wty;
    s.yty = yty;
    s.n = n;
    return s;
  }
};

// ---------------------------------------------------------------- kernels.cpp:43-55
double eval_kernel(const Vec& ls, double outputscale, const Vec& x, const Vec& x2) {
  double q = 0.0;
  for (std::size_t i = 0; i < x.size(); ++i) {
    const double d = (x[i] - x2[i]) / ls[i];
    q += d * d;
  }
  return outputscale * std::exp(-0.5 * q);
}

// ---------------------------------------------------------------- grid.cpp:73-82
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

// Mixed-radix complex FFT (stand-in for FFTW; the transform sizes are 5-smooth).
struct FFT1 {
  std::size_t n = 1;
  std::vector<int> factors;
  std::vector<cplx> tw;  // tw[j] = exp(-2 pi i j / n)
  explicit FFT1(std::size_t n_) : n(n_) {
    std::size_t r = n;
    for (int f : {4, 2, 3, 5}) {
      while (r % f == 0) {
        factors.push_back(f);
        r /= f;
      }
    }
    if (r != 1) factors.push_back(static_cast<int>(r));  // generic DFT radix
    tw.resize(n);
    for (std::size_t j = 0; j < n; ++j) {
      const double ang = -2.0 * M_PI * static_cast<double>(j) / static_cast<double>(n);
      tw[j] = cplx(std::cos(ang), std::sin(ang));
    }
  }
  cplx w(std::size_t j, bool inv) const {
    const cplx v = tw[j % n];
    return inv ? std::conj(v) : v;
  }
  void rec(const cplx* in, std::size_t istride, cplx* out, std::size_t len, std::size_t fi,
           std::size_t twstride, bool inv) const {
    if (len == 1) {
      out[0] = in[0];
      return;
    }
    const std::size_t r = static_cast<std::size_t>(factors[fi]);
    const std::size_t m = len / r;
    for (std::size_t q = 0; q < r; ++q) {
      rec(in + q * istride, istride * r, out + q * m, m, fi + 1, twstride * r, inv);
    }
    cplx t[64];
    cplx acc[64];
    for (std::size_t k = 0; k < m; ++k) {
      for (std::size_t q = 0; q < r; ++q) t[q] = out[q * m + k] * w(q * k * twstride, inv);
      for (std::size_t s = 0; s < r; ++s) {
        cplx a(0.0, 0.0);
        for (std::size_t q = 0; q < r; ++q) a += t[q] * w(q * s * m * twstride, inv);
        acc[s] = a;
      }
      for (std::size_t s = 0; s < r; ++s) out[k + s * m] = acc[s];
    }
  }
  void run(const cplx* in, cplx* out, bool inv) const { rec(in, 1, out, n, 0, 1, inv); }
};

struct FFTN {
  std::vector<std::size_t> shape;
  std::vector<FFT1> plans;
  std::size_t total = 1;
  explicit FFTN(const std::vector<std::size_t>& s) : shape(s) {
    for (std::size_t e : s) {
      plans.emplace_back(e);
      total *= e;
    }
  }
  void run(std::vector<cplx>& a, bool inv) const {
    const std::size_t d = shape.size();
    std::size_t inner = total;
    for (std::size_t k = 0; k < d; ++k) {
      const std::size_t len = shape[k];
      inner /= len;
      const std::size_t outer = total / (len * inner);
      par_for(static_cast<int64_t>(outer * inner), [&](int64_t lo, int64_t hi) {
        std::vector<cplx> line(len), res(len);
        for (int64_t li = lo; li < hi; ++li) {
          const std::size_t o = static_cast<std::size_t>(li) / inner;
          const std::size_t i = static_cast<std::size_t>(li) % inner;
          const std::size_t base = o * len * inner + i;
          for (std::size_t j = 0; j < len; ++j) line[j] = a[base + j * inner];
          plans[k].run(line.data(), res.data(), inv);
          for (std::size_t j = 0; j < len; ++j) a[base + j * inner] = res[j];
        }
      });
    }
  }
};

// ---------------------------------------------------------------- grid.cpp:94-151,193-235
struct Toeplitz {
  Grid grid;
  Vec ls;
  double outputscale = 1.0;
  double sigma_sq = 0.0;
  std::vector<int64_t> shape, embed_shape;
  std::size_t embed_total = 0;
  std::vector<cplx> spectrum;
  FFTN* fft = nullptr;

  Vec generator() const {  // grid.cpp:42-52
    const Vec origin = grid.point(0);
    Vec t(grid.m);
    for (int64_t j = 0; j < grid.m; ++j) t[j] = eval_kernel(ls, outputscale, origin, grid.point(j));
    return t;
  }

  Toeplitz(const Grid& g, const Vec& ls_, double os, double noise_std)
      : grid(g), ls(ls_), outputscale(os), sigma_sq(noise_std * noise_std) {
    const int d = grid.d;
    shape.resize(d);
    embed_shape.resize(d);
    embed_total = 1;
    std::vector<std::size_t> es(d);
    for (int k = 0; k < d; ++k) {
      shape[k] = grid.sz[k];
      embed_shape[k] = next_fast_fft_size(2 * shape[k] - 1);
      embed_total *= static_cast<std::size_t>(embed_shape[k]);
      es[k] = static_cast<std::size_t>(embed_shape[k]);
    }
    const Vec gen = generator();
    std::vector<cplx> embed(embed_total, cplx(0.0, 0.0));
    std::vector<int64_t> idx(d, 0);
    for (std::size_t flat = 0; flat < embed_total; ++flat) {
      int64_t gen_flat = 0;
      bool in_support = true;
      for (int k = 0; k < d && in_support; ++k) {
        int64_t delta;
        if (idx[k] < shape[k]) {
          delta = idx[k];
        } else if (embed_shape[k] - idx[k] < shape[k]) {
          delta = embed_shape[k] - idx[k];
        } else {
          in_support = false;
          delta = 0;
        }
        gen_flat = gen_flat * shape[k] + delta;
      }
      if (in_support) embed[flat] = cplx(gen[gen_flat], 0.0);
      for (int k = d - 1; k >= 0; --k) {
        if (++idx[k] < embed_shape[k]) break;
        idx[k] = 0;
      }
    }
    fft = new FFTN(es);
    fft->run(embed, false);
    spectrum = std::move(embed);
  }
  ~Toeplitz() { delete fft; }

  // Sensitivity-study mode (orc_kg_set_direct): K_G v as d direct Toeplitz mode products
  // (K_G = T_0 ⊗ … ⊗ T_{d-1} for the separable SE kernel, kernels.cpp:43-55), summed in
  // index order.  Same operator as the circulant FFT below up to rounding — a second valid
  // rounding of the reference's math, used to measure how far CG traces and iteration counts
  // move under O(1e-16) perturbations of K_G.  Not the reference's algorithm.
  bool direct = false;
  Vec apply_direct(const Vec& v) const {
    const int d = grid.d;
    Vec cur = v, nxt(grid.m);
    int64_t inner = grid.m;
    for (int k = 0; k < d; ++k) {
      const int64_t len = shape[k];
      inner /= len;
      const int64_t outer = grid.m / (len * inner);
      const double h = grid.sp[k];
      Vec gen(len);
      for (int64_t j = 0; j < len; ++j) {
        const double q = static_cast<double>(j) * h / ls[k];
        gen[j] = std::exp(-0.5 * q * q) * (k == 0 ? outputscale : 1.0);
      }
      par_for(outer * inner, [&](int64_t lo, int64_t hi) {
        for (int64_t li = lo; li < hi; ++li) {
          const int64_t o = li / inner, i = li % inner;
          const int64_t base = o * len * inner + i;
          for (int64_t a = 0; a < len; ++a) {
            double s = 0.0;
            for (int64_t j = 0; j < len; ++j) s += gen[a > j ? a - j : j - a] * cur[base + j * inner];
            nxt[base + a * inner] = s;
          }
        }
      });
      std::swap(cur, nxt);
    }
    return cur;
  }

  std::size_t eflat_of(int64_t flat) const {
    std::size_t e = 0;
    std::vector<int64_t> idx(grid.d);
    for (int k = grid.d - 1; k >= 0; --k) {
      idx[k] = flat % shape[k];
      flat /= shape[k];
    }
    for (int k = 0; k < grid.d; ++k) e = e * embed_shape[k] + idx[k];
    return e;
  }

  Vec apply(const Vec& v) const {
    if (static_cast<int64_t>(v.size()) != grid.m) {
      throw std::invalid_argument("ToeplitzOperator::apply: length mismatch");
    }
    if (direct) return apply_direct(v);
    std::vector<cplx> buf(embed_total, cplx(0.0, 0.0));
    const int d = grid.d;
    std::vector<int64_t> idx(d, 0);
    std::vector<std::size_t> emap(grid.m);
    for (int64_t flat = 0; flat < grid.m; ++flat) {
      std::size_t eflat = 0;
      for (int k = 0; k < d; ++k) eflat = eflat * embed_shape[k] + idx[k];
      emap[flat] = eflat;
      buf[eflat] = cplx(v[flat], 0.0);
      for (int k = d - 1; k >= 0; --k) {
        if (++idx[k] < shape[k]) break;
        idx[k] = 0;
      }
    }
    fft->run(buf, false);
    for (std::size_t i = 0; i < embed_total; ++i) buf[i] *= spectrum[i];
    fft->run(buf, true);
    const double scale = 1.0 / static_cast<double>(embed_total);
    Vec out(grid.m);
    for (int64_t flat = 0; flat < grid.m; ++flat) out[flat] = buf[emap[flat]].real() * scale;
    return out;
  }
};

// ---------------------------------------------------------------- vector helpers
double dot(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

// ---------------------------------------------------------------- solvers.cpp:271-336
struct GridSolveResult {
  Vec xhat_d;
  int iterations = 0;
  bool converged = false;
  double residual_sq = 0.0;
  Vec residual_trace, alphas, betas;
  double loop_seconds = 0.0;
};

GridSolveResult factorized_cg_grid_rhs(const Toeplitz& kg, const Stats& stats, const Vec& rhat0,
                                       double sigma, double eps_abs, double rel_tol,
                                       int maxiter) {
  const int64_t m = kg.grid.m;
  if (static_cast<int64_t>(rhat0.size()) != m) {
    throw std::invalid_argument("factorized_cg_grid_rhs: dimension mismatch");
  }
  if (eps_abs < 0.0 && rel_tol < 0.0) {
    throw std::invalid_argument("factorized_cg_grid_rhs: set eps_abs or rel_tol");
  }
  GridSolveResult res;
  const double sigma_sq = sigma * sigma;
  Vec rhat = rhat0;
  Vec uhat = stats.apply_wtw(rhat);
  Vec vhat = kg.apply(uhat);
  for (int64_t i = 0; i < m; ++i) vhat[i] += sigma_sq * rhat[i];
  Vec shat = uhat;
  Vec zbar = vhat;
  Vec xhat_d(m, 0.0);
  double rho = dot(uhat, rhat);
  const double eps = eps_abs >= 0.0 ? eps_abs : rel_tol * rel_tol * rho;
  res.residual_trace.push_back(rho);
  if (rho <= eps) {
    res.xhat_d = std::move(xhat_d);
    res.converged = true;
    res.residual_sq = rho;
    return res;
  }
  const auto t1 = std::chrono::steady_clock::now();
  for (int k = 0; k < maxiter; ++k) {
    const double pap = dot(shat, zbar);
    if (pap <= 0.0) {
      throw SolverBreakdown(
          "factorized_cg_grid_rhs: p^T A p <= 0, operator is not positive definite");
    }
    const double alpha = rho / pap;
    for (int64_t i = 0; i < m; ++i) xhat_d[i] += alpha * shat[i];
    for (int64_t i = 0; i < m; ++i) rhat[i] -= alpha * zbar[i];
    uhat = stats.apply_wtw(rhat);
    vhat = kg.apply(uhat);
    for (int64_t i = 0; i < m; ++i) vhat[i] += sigma_sq * rhat[i];
    const double rho_new = dot(uhat, rhat);
    res.iterations = k + 1;
    res.alphas.push_back(alpha);
    res.residual_trace.push_back(rho_new);
    if (rho_new <= eps) {
      res.converged = true;
      rho = rho_new;
      break;
    }
    const double beta = rho_new / rho;
    res.betas.push_back(beta);
    for (int64_t i = 0; i < m; ++i) shat[i] = uhat[i] + beta * shat[i];
    for (int64_t i = 0; i < m; ++i) zbar[i] = vhat[i] + beta * zbar[i];
    rho = rho_new;
  }
  res.loop_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
  res.xhat_d = std::move(xhat_d);
  res.residual_sq = rho;
  return res;
}

// gp.cpp:326-352
Vec posterior_mean_gsgp(const Toeplitz& kg, const Stats& stats, double sigma, double tol,
                        int maxiter, int* iterations, double* residual_sq) {
  const double sigma_sq = sigma * sigma;
  Vec rhat0 = kg.apply(stats.wty);
  for (auto& v : rhat0) v = -v / sigma_sq;
  const double eps_abs = tol * tol * stats.yty;
  const GridSolveResult solve =
      factorized_cg_grid_rhs(kg, stats, rhat0, sigma, eps_abs, -1.0, maxiter);
  if (!solve.converged) {
    throw SolverNonConvergence("posterior_mean_gsgp: solver hit maxiter", solve.residual_sq,
                               solve.iterations);
  }
  Vec rhs(kg.grid.m);
  for (int64_t i = 0; i < kg.grid.m; ++i) rhs[i] = solve.xhat_d[i] + stats.wty[i] / sigma_sq;
  if (iterations) *iterations = solve.iterations;
  if (residual_sq) *residual_sq = solve.residual_sq;
  return kg.apply(rhs);
}

// ---------------------------------------------------------------- gp.cpp:16-25
Vec rademacher_probe(int64_t dim, uint64_t seed, uint64_t probe_index) {
  std::seed_seq seq{static_cast<std::uint32_t>(seed), static_cast<std::uint32_t>(seed >> 32),
                    static_cast<std::uint32_t>(probe_index),
                    static_cast<std::uint32_t>(probe_index >> 32)};
  std::mt19937_64 rng(seq);
  Vec v(dim);
  for (int64_t i = 0; i < dim; ++i) v[i] = (rng() & 1) ? 1.0 : -1.0;
  return v;
}

// Symmetric tridiagonal eigensolver (implicit QL with Wilkinson-type shifts) tracking the
// first row of the eigenvector matrix — what quadrature_logdet reads from Eigen's
// SelfAdjointEigenSolver::computeFromTridiagonal (gp.cpp:38-56).  Eigenvalues ascending.
void tridiag_eig(int n, const double* alpha, const double* beta, Vec& dd, Vec& z) {
  dd.assign(alpha, alpha + n);
  Vec e(n, 0.0);
  for (int i = 0; i + 1 < n; ++i) e[i] = beta[i];
  z.assign(n, 0.0);
  z[0] = 1.0;
  for (int l = 0; l < n; ++l) {
    int iter = 0;
    int mm;
    do {
      for (mm = l; mm < n - 1; ++mm) {
        const double s = std::abs(dd[mm]) + std::abs(dd[mm + 1]);
        if (std::abs(e[mm]) <= std::numeric_limits<double>::epsilon() * s) break;
      }
      if (mm != l) {
        if (++iter > 200) throw std::runtime_error("tridiag_eig: no convergence");
        double g = (dd[l + 1] - dd[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = dd[mm] - dd[l] + e[l] / (g + std::copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        bool early = false;
        for (i = mm - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = std::hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            dd[i + 1] -= p;
            e[mm] = 0.0;
            early = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = dd[i + 1] - p;
          r = (dd[i] - g) * s + 2.0 * c * b;
          p = s * r;
          dd[i + 1] = g + p;
          g = c * r - b;
          f = z[i + 1];
          z[i + 1] = s * z[i] + c * f;
          z[i] = c * z[i] - s * f;
        }
        if (early) continue;
        dd[l] -= p;
        e[l] = g;
        e[mm] = 0.0;
      }
    } while (mm != l);
  }
  std::vector<int> ord(n);
  for (int i = 0; i < n; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return dd[a] < dd[b]; });
  Vec d2(n), z2(n);
  for (int i = 0; i < n; ++i) {
    d2[i] = dd[ord[i]];
    z2[i] = z[ord[i]];
  }
  dd.swap(d2);
  z.swap(z2);
}

// gp.cpp:34-63
std::pair<double, int> quadrature_logdet(const Vec& alpha, const Vec& beta, double probe_sq,
                                         double quad_tol) {
  const int k = static_cast<int>(alpha.size());
  double prev = 0.0;
  double value = 0.0;
  int depth = 0;
  Vec lam, z;
  for (int j = 1; j <= k; ++j) {
    tridiag_eig(j, alpha.data(), beta.data(), lam, z);
    double mx = 0.0;
    for (double v : lam) mx = std::max(mx, std::abs(v));
    const double scale = std::max(mx, 1e-300);
    if (lam[0] < -1e-10 * scale) {
      throw std::runtime_error(
          "slq_logdet: negative Ritz value, operator is not positive definite");
    }
    double est = 0.0;
    for (int l = 0; l < j; ++l) {
      const double tau = z[l];
      est += tau * tau * std::log(std::max(lam[l], 1e-16 * scale));
    }
    est *= probe_sq;
    value = est;
    depth = j;
    if (j >= 2 && quad_tol > 0.0 &&
        std::abs(est - prev) <= quad_tol * std::max(std::abs(est), 1e-300)) {
      break;
    }
    prev = est;
  }
  return {value, depth};
}

// ---------------------------------------------------------------- solvers.cpp:464-538
struct Tridiag {
  Vec alpha, beta, d;
  std::vector<Vec> basis;  // columns
};

Tridiag factorized_lanczos_fused(const Toeplitz& kg, const Stats& stats, const Vec& kgwt_z0_in,
                                 const Vec& wt_z0_in, double z0_sq, double sigma_sq, int k,
                                 bool keep_basis) {
  const int64_t m = kg.grid.m;
  if (k < 1) throw std::invalid_argument("factorized_lanczos_fused: bad k");
  if (z0_sq <= 0.0) throw std::invalid_argument("factorized_lanczos_fused: start vector is zero");
  const double bnorm = std::sqrt(z0_sq);
  Vec wt_z0(m), kgwt_z0(m);
  for (int64_t i = 0; i < m; ++i) {
    wt_z0[i] = wt_z0_in[i] / bnorm;
    kgwt_z0[i] = kgwt_z0_in[i] / bnorm;
  }
  std::vector<Vec> qhat(k, Vec(m, 0.0));
  std::vector<Vec> phat(k, Vec(m, 0.0));
  Vec d(k, 0.0), tq(k, 0.0), alpha(k, 0.0), beta(k > 1 ? k - 1 : 0, 0.0);
  Vec q(m, 0.0), q_prev(m, 0.0), sbar(m, 0.0), pcur(m, 0.0);
  double cq = 1.0, cq_prev = 0.0;
  d[0] = cq;
  double beta_prev = 0.0, scale = 0.0;
  int done = k;
  Vec wv(m);
  for (int i = 0; i < k; ++i) {
    for (int64_t r = 0; r < m; ++r) wv[r] = sbar[r] + cq * kgwt_z0[r] - beta_prev * q_prev[r];
    double e = sigma_sq * cq - beta_prev * cq_prev;
    alpha[i] = dot(pcur, wv) + e * tq[i] + cq * dot(wv, wt_z0) + cq * e;
    scale = std::max(scale, std::abs(alpha[i]));
    if (i == k - 1) break;
    for (int64_t r = 0; r < m; ++r) wv[r] -= alpha[i] * q[r];
    e -= alpha[i] * cq;
    const double wdot = dot(wv, wt_z0);
    Vec lambda(i + 1);
    for (int j = 0; j <= i; ++j) lambda[j] = dot(phat[j], wv) + e * tq[j] + (wdot + e) * d[j];
    for (int j = 0; j <= i; ++j) {
      for (int64_t r = 0; r < m; ++r) wv[r] -= qhat[j][r] * lambda[j];
    }
    double dl = 0.0;
    for (int j = 0; j <= i; ++j) dl += d[j] * lambda[j];
    e -= dl;
    const Vec p_next = stats.apply_wtw(wv);
    Vec s_next = kg.apply(p_next);
    for (int64_t r = 0; r < m; ++r) s_next[r] += sigma_sq * wv[r];
    const double b_next =
        std::sqrt(std::max(0.0, dot(p_next, wv) + 2.0 * e * dot(wv, wt_z0) + e * e));
    if (b_next <= 1e-12 * std::max(scale, 1e-300)) {
      done = i + 1;
      break;
    }
    beta[i] = b_next;
    scale = std::max(scale, b_next);
    q_prev = q;
    cq_prev = cq;
    for (int64_t r = 0; r < m; ++r) {
      q[r] = wv[r] / b_next;
      pcur[r] = p_next[r] / b_next;
      sbar[r] = s_next[r] / b_next;
    }
    cq = e / b_next;
    qhat[i + 1] = q;
    phat[i + 1] = pcur;
    d[i + 1] = cq;
    tq[i + 1] = dot(q, wt_z0);
    beta_prev = b_next;
  }
  Tridiag out;
  out.alpha.assign(alpha.begin(), alpha.begin() + done);
  out.beta.assign(beta.begin(), beta.begin() + (done > 1 ? done - 1 : 0));
  out.d.assign(d.begin(), d.begin() + done);
  if (keep_basis) out.basis.assign(qhat.begin(), qhat.begin() + done);
  return out;
}

// W^T u as a stream over the points (InterpMatrix::apply_transpose, interp.cpp:145-151:
// Eigen's transpose product visits rows in order, so the accumulation order matches).
Vec wt_apply(const Grid& grid, int scheme, const double* x, int64_t n, const Vec& u) {
  Vec out(grid.m, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    const WeightVector w = interp_weights(grid, x + i * grid.d, scheme);
    for (std::size_t a = 0; a < w.indices.size(); ++a) out[w.indices[a]] += w.values[a] * u[i];
  }
  return out;
}

// gp.cpp:85-111 (W^T v streamed instead of a materialised W)
std::pair<double, int> slq_logdet_ski_factorized(const Toeplitz& kg, const Stats& stats,
                                                 const Grid& grid, int scheme, const double* x,
                                                 int64_t n, double sigma, int num_probes,
                                                 int max_depth, double quad_tol, uint64_t seed) {
  if (num_probes < 1) {
    throw std::invalid_argument("slq_logdet_ski_factorized: need at least one probe");
  }
  const int depth = static_cast<int>(std::min<int64_t>(max_depth, n));
  // probes are independent (gp.cpp:94-108); they run on the host threads and are summed in
  // probe order afterwards, as the reference's sequential loop does
  std::vector<std::pair<double, int>> per(num_probes);
  std::vector<std::exception_ptr> errs(num_probes);
  par_for(num_probes, [&](int64_t lo, int64_t hi) {
    for (int64_t p = lo; p < hi; ++p) {
      try {
        const Vec v = rademacher_probe(n, seed, static_cast<uint64_t>(p));
        const Vec wt = wt_apply(grid, scheme, x, n, v);
        const Vec kgwt = kg.apply(wt);
        const double z0_sq = dot(v, v);
        const Tridiag t =
            factorized_lanczos_fused(kg, stats, kgwt, wt, z0_sq, sigma * sigma, depth, false);
        per[p] = quadrature_logdet(t.alpha, t.beta, z0_sq, quad_tol);
      } catch (...) {
        errs[p] = std::current_exception();
      }
    }
  }, 1);
  double total = 0.0;
  int max_used = 0;
  for (int p = 0; p < num_probes; ++p) {
    if (errs[p]) std::rethrow_exception(errs[p]);
    total += per[p].first;
    max_used = std::max(max_used, per[p].second);
  }
  return {total / num_probes, max_used};
}

// solvers.cpp:351-389 — Lanczos with full reorthogonalisation on an m-dim operator.
template <class Op>
std::pair<Vec, Vec> lanczos(const Op& op, int64_t n, const Vec& b, int k) {
  if (k < 1 || k > n) throw std::invalid_argument("lanczos: need 1 <= k <= dim");
  const double bnorm = std::sqrt(dot(b, b));
  if (bnorm == 0.0) throw std::invalid_argument("lanczos: start vector is zero");
  std::vector<Vec> q(k, Vec(n, 0.0));
  Vec alpha(k, 0.0), beta(k > 1 ? k - 1 : 0, 0.0);
  for (int64_t i = 0; i < n; ++i) q[0][i] = b[i] / bnorm;
  double beta_prev = 0.0, scale = 0.0;
  int done = k;
  for (int i = 0; i < k; ++i) {
    Vec w = op(q[i]);
    if (i > 0) {
      for (int64_t r = 0; r < n; ++r) w[r] -= beta_prev * q[i - 1][r];
    }
    alpha[i] = dot(q[i], w);
    scale = std::max(scale, std::abs(alpha[i]));
    if (i == k - 1) break;
    for (int64_t r = 0; r < n; ++r) w[r] -= alpha[i] * q[i][r];
    Vec c(i + 1);
    for (int j = 0; j <= i; ++j) c[j] = dot(q[j], w);
    for (int j = 0; j <= i; ++j) {
      for (int64_t r = 0; r < n; ++r) w[r] -= q[j][r] * c[j];
    }
    const double b_next = std::sqrt(dot(w, w));
    if (b_next <= 1e-12 * std::max(scale, 1e-300)) {
      done = i + 1;
      break;
    }
    beta[i] = b_next;
    scale = std::max(scale, b_next);
    for (int64_t r = 0; r < n; ++r) q[i + 1][r] = w[r] / b_next;
    beta_prev = b_next;
  }
  alpha.resize(done);
  beta.resize(done > 1 ? done - 1 : 0);
  return {alpha, beta};
}

// gp.cpp:67-83
template <class Op>
double slq_logdet(const Op& op, int64_t dim, int num_probes, int max_depth, double quad_tol,
                  uint64_t seed) {
  if (num_probes < 1) throw std::invalid_argument("slq_logdet: need at least one probe");
  const int depth = static_cast<int>(std::min<int64_t>(max_depth, dim));
  double total = 0.0;
  for (int p = 0; p < num_probes; ++p) {
    const Vec v = rademacher_probe(dim, seed, p);
    const auto t = lanczos(op, dim, v, depth);
    total += quadrature_logdet(t.first, t.second, dot(v, v), quad_tol).first;
  }
  return total / num_probes;
}

// gp.cpp:142-154
double estimate_grid_kernel_condition(const Toeplitz& kg) {
  const int64_t m = kg.grid.m;
  const int depth = static_cast<int>(std::min<int64_t>(30, m));
  const Vec v = rademacher_probe(m, 0x5eedf00d, 0);
  const auto t = lanczos([&](const Vec& u) { return kg.apply(u); }, m, v, depth);
  Vec lam, z;
  tridiag_eig(static_cast<int>(t.first.size()), t.first.data(), t.second.data(), lam, z);
  const double hi = lam.back();
  const double lo = lam.front();
  if (!(hi > 0.0)) return std::numeric_limits<double>::infinity();
  return hi / std::max(lo, hi * 1e-18);
}

// gp.cpp:116-140 — dense LU of K_G W^T W + sigma^2 I (partial pivoting).
double dense_logdet_grid_system(const Toeplitz& kg, const Stats& stats, double sigma_sq) {
  const int64_t m = kg.grid.m;
  std::vector<Vec> kcols(m);
  Vec e(m, 0.0);
  for (int64_t j = 0; j < m; ++j) {
    e[j] = 1.0;
    kcols[j] = kg.apply(e);
    e[j] = 0.0;
  }
  // sys = K * WtW, row-major a[i*m+j] = sum_l K(i,l) WtW(l,j)
  Vec a(m * m, 0.0);
  for (int64_t l = 0; l < m; ++l) {
    for (int64_t kk = stats.row_ptr[l]; kk < stats.row_ptr[l + 1]; ++kk) {
      const int64_t j = stats.col[kk];
      const double v = stats.val[kk];
      for (int64_t i = 0; i < m; ++i) a[i * m + j] += kcols[l][i] * v;
    }
  }
  for (int64_t i = 0; i < m; ++i) a[i * m + i] += sigma_sq;
  double logdet = 0.0;
  for (int64_t c = 0; c < m; ++c) {
    int64_t piv = c;
    for (int64_t r = c + 1; r < m; ++r) {
      if (std::abs(a[r * m + c]) > std::abs(a[piv * m + c])) piv = r;
    }
    if (piv != c) {
      for (int64_t j = 0; j < m; ++j) std::swap(a[c * m + j], a[piv * m + j]);
    }
    const double dg = a[c * m + c];
    logdet += std::log(std::abs(dg));
    if (dg == 0.0) continue;
    for (int64_t r = c + 1; r < m; ++r) {
      const double f = a[r * m + c] / dg;
      if (f == 0.0) continue;
      for (int64_t j = c + 1; j < m; ++j) a[r * m + j] -= f * a[c * m + j];
    }
  }
  return logdet;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return ORC_OK;
  } catch (const OutOfGrid& e) {
    g_err = e.what();
    return ORC_OUT_OF_GRID;
  } catch (const SolverBreakdown& e) {
    g_err = e.what();
    return ORC_BREAKDOWN;
  } catch (const SolverNonConvergence& e) {
    g_err = e.what();
    return ORC_NONCONVERGENCE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ORC_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ORC_RUNTIME_ERROR;
  }
}

template <class T>
Stats run_stats(const Grid& grid, int scheme, const T* x, const T* y, int64_t n, int nthreads) {
  const int d = grid.d;
  if (nthreads < 1) nthreads = 1;
  if (n < 1024 * nthreads) nthreads = 1;
  std::vector<Accumulator*> accs(nthreads, nullptr);
  std::vector<int64_t> bad_row(nthreads, -1);
  std::vector<std::string> bad_msg(nthreads);
  auto work = [&](int t) {
    const int64_t lo = n * t / nthreads, hi = n * (t + 1) / nthreads;
    accs[t] = new Accumulator(grid, scheme);
    std::vector<double> xv(d);
    for (int64_t i = lo; i < hi; ++i) {
      for (int k = 0; k < d; ++k) xv[k] = static_cast<double>(x[i * d + k]);
      try {
        accs[t]->add(xv.data(), static_cast<double>(y[i]));
      } catch (const OutOfGrid& e) {
        bad_row[t] = i + 1;
        bad_msg[t] = e.what();
        return;
      }
    }
  };
  if (nthreads == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) th.emplace_back(work, t);
    for (auto& h : th) h.join();
  }
  for (int t = 0; t < nthreads; ++t) {
    if (bad_row[t] >= 0) {
      for (auto* a : accs) delete a;
      g_err_row = bad_row[t];
      throw OutOfGrid("sufficient_stats: stream row " + std::to_string(bad_row[t]) + ": " +
                      bad_msg[t]);
    }
  }
  // merge() (interp.cpp:202-210) as a pairwise tree over the shards, independent pairs on
  // their own threads (a sum, so only the order of the hash-map additions changes)
  for (int stride = 1; stride < nthreads; stride *= 2) {
    std::vector<std::thread> th;
    for (int t = 0; t + stride < nthreads; t += 2 * stride) {
      th.emplace_back([&, t, stride] { accs[t]->merge(*accs[t + stride]); });
    }
    for (auto& h : th) h.join();
  }
  Stats s = accs[0]->finalize();
  for (auto* a : accs) delete a;
  return s;
}

// ---------------------------------------------------------------- gp.cpp:381-427
// posterior_cov_exact: one grid-rhs EFCG per test point (rel_tol = tol), then
// cov(i, j) = w_iᵀ h_j − h_i · x̂_j with h_j = K_G w_j; returns the symmetrised matrix.
struct CovOut {
  Vec cov;
  double max_asymmetry = 0.0;
  int total_iterations = 0;
};

CovOut posterior_cov_exact(const Toeplitz& kg, const Stats& stats, int scheme, double sigma, const double* pts,
                           int64_t ns, double tol, int maxiter) {
  const int64_t m = kg.grid.m;
  const int d = kg.grid.d;
  std::vector<WeightVector> wx(ns);
  std::vector<Vec> h(ns);
  for (int64_t j = 0; j < ns; ++j) {
    wx[j] = interp_weights(kg.grid, pts + j * d, scheme);
    Vec dense(m, 0.0);
    for (std::size_t a = 0; a < wx[j].indices.size(); ++a) dense[wx[j].indices[a]] = wx[j].values[a];
    h[j] = kg.apply(dense);
  }
  CovOut res;
  std::vector<Vec> solved(ns);
  for (int64_t j = 0; j < ns; ++j) {
    const GridSolveResult s = factorized_cg_grid_rhs(kg, stats, h[j], sigma, -1.0, tol, maxiter);
    if (!s.converged) {
      throw SolverNonConvergence("posterior_cov_exact: solver hit maxiter", s.residual_sq, s.iterations);
    }
    res.total_iterations += s.iterations;
    solved[j] = s.xhat_d;
  }
  Vec cov(ns * ns);
  for (int64_t i = 0; i < ns; ++i) {
    for (int64_t j = 0; j < ns; ++j) {
      double prior = 0.0;
      for (std::size_t a = 0; a < wx[i].indices.size(); ++a) prior += wx[i].values[a] * h[j][wx[i].indices[a]];
      cov[i * ns + j] = prior - dot(h[i], solved[j]);
    }
  }
  res.cov.assign(ns * ns, 0.0);
  for (int64_t i = 0; i < ns; ++i) {
    for (int64_t j = 0; j < ns; ++j) {
      res.max_asymmetry = std::max(res.max_asymmetry, std::abs(cov[i * ns + j] - cov[j * ns + i]));
      res.cov[i * ns + j] = 0.5 * (cov[i * ns + j] + cov[j * ns + i]);
    }
  }
  return res;
}

// ---------------------------------------------------------------- gp.cpp:429-528
// posterior_cov_lowrank: EFLA from ĝ = WᵀW 1 / ‖·‖ with the basis kept;
// R[:, j] = K_G (WᵀW q̂_j + d_j WᵀW ĝ / √(ĝᵀWᵀWĝ)), T = tridiag(α, β).
struct LowRank {
  int64_t m = 0;
  int k = 0;
  std::vector<Vec> r;  // columns
  Vec alpha, beta;
};

LowRank posterior_cov_lowrank(const Toeplitz& kg, const Stats& stats, double sigma, int64_t rank) {
  const int64_t m = kg.grid.m;
  if (rank < 0 || rank > m) throw std::invalid_argument("posterior_cov_lowrank: need 0 <= rank <= grid size");
  LowRank out;
  out.m = m;
  if (rank == 0 || stats.n == 0) return out;
  const Vec g_raw = stats.apply_wtw(Vec(m, 1.0));
  const double g_norm = std::sqrt(dot(g_raw, g_raw));
  if (g_norm == 0.0) return out;
  Vec ghat(m);
  for (int64_t i = 0; i < m; ++i) ghat[i] = g_raw[i] / g_norm;
  const Vec wt_z0 = stats.apply_wtw(ghat);
  const Vec kgwt_z0 = kg.apply(wt_z0);
  const double z0_sq = dot(ghat, wt_z0);
  if (z0_sq <= 0.0) return out;
  const Tridiag f = factorized_lanczos_fused(kg, stats, kgwt_z0, wt_z0, z0_sq, sigma * sigma,
                                             static_cast<int>(rank), true);
  const int k = static_cast<int>(f.alpha.size());
  const double bn = std::sqrt(z0_sq);
  out.k = k;
  out.alpha = f.alpha;
  out.beta = f.beta;
  for (int j = 0; j < k; ++j) {
    Vec u = stats.apply_wtw(f.basis[j]);
    for (int64_t i = 0; i < m; ++i) u[i] += f.d[j] * (wt_z0[i] / bn);
    out.r.push_back(kg.apply(u));
  }
  return out;
}

// T x = b for the symmetric tridiagonal T (LDLᵀ without pivoting; T is positive definite
// for a positive definite operator — Eigen's LDLT agrees to rounding).
Vec tridiag_solve(const Vec& a, const Vec& b_off, const Vec& rhs) {
  const int k = static_cast<int>(a.size());
  Vec dd(k), l(k > 1 ? k - 1 : 0), z(rhs);
  dd[0] = a[0];
  for (int i = 1; i < k; ++i) {
    l[i - 1] = b_off[i - 1] / dd[i - 1];
    dd[i] = a[i] - l[i - 1] * b_off[i - 1];
  }
  for (int i = 1; i < k; ++i) z[i] -= l[i - 1] * z[i - 1];
  for (int i = 0; i < k; ++i) z[i] /= dd[i];
  for (int i = k - 2; i >= 0; --i) z[i] -= l[i] * z[i + 1];
  return z;
}

Vec lowrank_phi(const LowRank& lr, const WeightVector& w) {
  Vec phi(lr.k, 0.0);
  for (std::size_t a = 0; a < w.indices.size(); ++a)
    for (int j = 0; j < lr.k; ++j) phi[j] += w.values[a] * lr.r[j][w.indices[a]];
  return phi;
}

// LowRankCov::cov_matrix (gp.cpp:500-525)
Vec lowrank_cov_matrix(const Toeplitz& kg, const LowRank& lr, int scheme, const double* pts, int64_t ns) {
  const int64_t m = kg.grid.m;
  const int d = kg.grid.d;
  std::vector<WeightVector> wx(ns);
  std::vector<Vec> h(ns);
  for (int64_t j = 0; j < ns; ++j) {
    wx[j] = interp_weights(kg.grid, pts + j * d, scheme);
    Vec dense(m, 0.0);
    for (std::size_t a = 0; a < wx[j].indices.size(); ++a) dense[wx[j].indices[a]] = wx[j].values[a];
    h[j] = kg.apply(dense);
  }
  Vec cov(ns * ns);
  for (int64_t i = 0; i < ns; ++i)
    for (int64_t j = 0; j < ns; ++j) {
      double prior = 0.0;
      for (std::size_t a = 0; a < wx[i].indices.size(); ++a) prior += wx[i].values[a] * h[j][wx[i].indices[a]];
      cov[i * ns + j] = prior;
    }
  if (lr.k > 0) {
    std::vector<Vec> phi(ns), tphi(ns);
    for (int64_t j = 0; j < ns; ++j) {
      phi[j] = lowrank_phi(lr, wx[j]);
      tphi[j] = tridiag_solve(lr.alpha, lr.beta, phi[j]);
    }
    for (int64_t i = 0; i < ns; ++i)
      for (int64_t j = 0; j < ns; ++j) cov[i * ns + j] -= dot(phi[i], tphi[j]);
  }
  Vec out(ns * ns);
  for (int64_t i = 0; i < ns; ++i)
    for (int64_t j = 0; j < ns; ++j) out[i * ns + j] = 0.5 * (cov[i * ns + j] + cov[j * ns + i]);
  return out;
}

// LowRankCov::query (gp.cpp:486-498)
double lowrank_query(const Toeplitz& kg, const LowRank& lr, int scheme, const double* x, const double* x2) {
  const int64_t m = kg.grid.m;
  const WeightVector wa = interp_weights(kg.grid, x, scheme);
  const WeightVector wb = interp_weights(kg.grid, x2, scheme);
  Vec dense(m, 0.0);
  for (std::size_t a = 0; a < wb.indices.size(); ++a) dense[wb.indices[a]] = wb.values[a];
  const Vec hb = kg.apply(dense);
  double prior = 0.0;
  for (std::size_t a = 0; a < wa.indices.size(); ++a) prior += wa.values[a] * hb[wa.indices[a]];
  if (lr.k == 0) return prior;
  const Vec pa = lowrank_phi(lr, wa), pb = lowrank_phi(lr, wb);
  return prior - dot(pa, tridiag_solve(lr.alpha, lr.beta, pb));
}

}  // namespace

struct orc_stats {
  Stats s;
};
struct orc_kg {
  Toeplitz* t;
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int64_t orc_last_error_row(void) { return g_err_row; }

int orc_fit_grid_to_data(int d, const double* lo, const double* hi, const int64_t* sizes,
                         int scheme, double* out_min, double* out_max) {
  return guard([&] {
    const int r = scheme == 0 ? 1 : 2;
    for (int k = 0; k < d; ++k) {
      const int64_t m = sizes[k];
      if (m < 2 * r + 2) {
        throw std::invalid_argument("fit_grid_to_data: need at least " +
                                    std::to_string(2 * r + 2) + " points per dimension");
      }
      if (!(hi[k] > lo[k])) throw std::invalid_argument("fit_grid_to_data: empty data range");
      const double s = (hi[k] - lo[k]) / static_cast<double>(m - 1 - 2 * r);
      out_min[k] = lo[k] - r * s;
      out_max[k] = hi[k] + r * s;
    }
  });
}

int orc_interp_weights(int d, const double* gmin, const double* gmax, const int64_t* gsize,
                       int scheme, const double* x, int64_t* idx, double* w, int* nnz) {
  return guard([&] {
    const Grid g(d, gmin, gmax, gsize);
    const WeightVector wv = interp_weights(g, x, scheme);
    for (std::size_t i = 0; i < wv.indices.size(); ++i) {
      idx[i] = wv.indices[i];
      w[i] = wv.values[i];
    }
    *nnz = static_cast<int>(wv.indices.size());
  });
}

int orc_sufficient_stats(int d, const double* gmin, const double* gmax, const int64_t* gsize,
                         int scheme, const double* x, const double* y, int64_t n,
                         int nthreads, orc_stats** out) {
  g_err_row = 0;
  return guard([&] {
    const Grid g(d, gmin, gmax, gsize);
    auto* h = new orc_stats{run_stats(g, scheme, x, y, n, nthreads)};
    *out = h;
  });
}

int orc_sufficient_stats_f32(int d, const double* gmin, const double* gmax,
                             const int64_t* gsize, int scheme, const float* x,
                             const float* y, int64_t n, int nthreads, orc_stats** out) {
  g_err_row = 0;
  return guard([&] {
    const Grid g(d, gmin, gmax, gsize);
    auto* h = new orc_stats{run_stats(g, scheme, x, y, n, nthreads)};
    *out = h;
  });
}

void orc_stats_destroy(orc_stats* s) { delete s; }

void orc_stats_info(const orc_stats* s, int64_t* m, int64_t* n, int64_t* nnz, double* yty) {
  *m = s->s.m;
  *n = s->s.n;
  *nnz = static_cast<int64_t>(s->s.val.size());
  *yty = s->s.yty;
}

void orc_stats_export(const orc_stats* s, int64_t* row_ptr, int64_t* col, double* val,
                      double* wty) {
  if (row_ptr) std::memcpy(row_ptr, s->s.row_ptr.data(), sizeof(int64_t) * (s->s.m + 1));
  if (col) std::memcpy(col, s->s.col.data(), sizeof(int64_t) * s->s.col.size());
  if (val) std::memcpy(val, s->s.val.data(), sizeof(double) * s->s.val.size());
  if (wty) std::memcpy(wty, s->s.wty.data(), sizeof(double) * s->s.m);
}

int orc_stats_from_csr(int64_t m, int64_t nnz, const int64_t* row_ptr, const int64_t* col,
                       const double* val, const double* wty, double yty, int64_t n,
                       orc_stats** out) {
  return guard([&] {
    auto* h = new orc_stats;
    h->s.m = m;
    h->s.row_ptr.assign(row_ptr, row_ptr + m + 1);
    h->s.col.assign(col, col + nnz);
    h->s.val.assign(val, val + nnz);
    h->s.wty.assign(wty, wty + m);
    h->s.yty = yty;
    h->s.n = n;
    *out = h;
  });
}

int orc_stats_apply_wtw(const orc_stats* s, const double* v, double* out) {
  return guard([&] {
    const Vec vv(v, v + s->s.m);
    const Vec r = s->s.apply_wtw(vv);
    std::memcpy(out, r.data(), sizeof(double) * s->s.m);
  });
}

int64_t orc_stats_max_row_nnz(const orc_stats* s) {  // interp.cpp:235-242
  int64_t best = 0;
  for (int64_t i = 0; i < s->s.m; ++i) {
    best = std::max(best, s->s.row_ptr[i + 1] - s->s.row_ptr[i]);
  }
  return best;
}

int orc_kg_create(int d, const double* gmin, const double* gmax, const int64_t* gsize,
                  const double* lengthscales, double outputscale, double noise_std,
                  orc_kg** out) {
  return guard([&] {
    const Grid g(d, gmin, gmax, gsize);
    const Vec ls(lengthscales, lengthscales + d);
    for (double l : ls) {
      if (!(l > 0.0)) throw std::invalid_argument("Hyperparams: lengthscales must be positive");
    }
    if (!(noise_std > 0.0)) throw std::invalid_argument("Hyperparams: noise_std must be positive");
    if (!(outputscale > 0.0)) {
      throw std::invalid_argument("Hyperparams: outputscale must be positive");
    }
    *out = new orc_kg{new Toeplitz(g, ls, outputscale, noise_std)};
  });
}

void orc_kg_destroy(orc_kg* k) {
  if (k) delete k->t;
  delete k;
}

int64_t orc_kg_dim(const orc_kg* k) { return k->t->grid.m; }

void orc_kg_embed_shape(const orc_kg* k, int64_t* shape) {
  for (int i = 0; i < k->t->grid.d; ++i) shape[i] = k->t->embed_shape[i];
}

int orc_kg_apply(const orc_kg* k, const double* v, double* out) {
  return guard([&] {
    const Vec vv(v, v + k->t->grid.m);
    const Vec r = k->t->apply(vv);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}

int orc_kernel_generator(const orc_kg* k, double* out) {
  return guard([&] {
    const Vec g = k->t->generator();
    std::memcpy(out, g.data(), sizeof(double) * g.size());
  });
}

int orc_kg_dense(const orc_kg* k, double* out, int64_t max_points) {  // grid.cpp:54-71
  return guard([&] {
    const Grid& grid = k->t->grid;
    const int64_t m = grid.m;
    if (m > max_points) {
      throw std::invalid_argument("kg_dense: grid has " + std::to_string(m) +
                                  " points, above the cap of " + std::to_string(max_points));
    }
    for (int64_t i = 0; i < m; ++i) {
      const Vec gi = grid.point(i);
      out[i * m + i] = k->t->outputscale;
      for (int64_t j = i + 1; j < m; ++j) {
        out[i * m + j] = eval_kernel(k->t->ls, k->t->outputscale, gi, grid.point(j));
        out[j * m + i] = out[i * m + j];
      }
    }
  });
}

int64_t orc_next_fast_fft_size(int64_t x) { return next_fast_fft_size(x); }

void orc_kg_set_direct(orc_kg* k, int direct) { k->t->direct = direct != 0; }

void orc_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int orc_get_threads(void) { return g_threads; }

int orc_factorized_cg_grid_rhs(const orc_kg* kg, const orc_stats* st, const double* rhat0,
                               double sigma, double eps_abs, double rel_tol, int maxiter,
                               double* xhat_d, int* iterations, int* converged,
                               double* residual_sq, double* residual_trace, double* alphas,
                               double* betas, double* loop_seconds) {
  return guard([&] {
    const Vec r0(rhat0, rhat0 + kg->t->grid.m);
    const GridSolveResult r =
        factorized_cg_grid_rhs(*kg->t, st->s, r0, sigma, eps_abs, rel_tol, maxiter);
    std::memcpy(xhat_d, r.xhat_d.data(), sizeof(double) * r.xhat_d.size());
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
    *residual_sq = r.residual_sq;
    if (residual_trace) {
      std::memcpy(residual_trace, r.residual_trace.data(), sizeof(double) * r.residual_trace.size());
    }
    if (alphas) std::memcpy(alphas, r.alphas.data(), sizeof(double) * r.alphas.size());
    if (betas) std::memcpy(betas, r.betas.data(), sizeof(double) * r.betas.size());
    if (loop_seconds) *loop_seconds = r.loop_seconds;
  });
}

int orc_posterior_mean_gsgp(const orc_kg* kg, const orc_stats* st, double sigma, double tol,
                            int maxiter, double* mean_coeffs, int* iterations,
                            double* residual_sq) {
  return guard([&] {
    const Vec mc = posterior_mean_gsgp(*kg->t, st->s, sigma, tol, maxiter, iterations,
                                       residual_sq);
    std::memcpy(mean_coeffs, mc.data(), sizeof(double) * mc.size());
  });
}

int orc_predict_mean(int d, const double* gmin, const double* gmax, const int64_t* gsize,
                     int scheme, const double* mean_coeffs, const double* pts, int64_t npts,
                     double* out) {
  return guard([&] {
    const Grid g(d, gmin, gmax, gsize);
    for (int64_t p = 0; p < npts; ++p) {
      const WeightVector wv = interp_weights(g, pts + p * d, scheme);
      double o = 0.0;
      for (std::size_t i = 0; i < wv.indices.size(); ++i) o += wv.values[i] * mean_coeffs[wv.indices[i]];
      out[p] = o;
    }
  });
}

void orc_rademacher_probe(int64_t n, uint64_t seed, uint64_t probe_index, double* out) {
  const Vec v = rademacher_probe(n, seed, probe_index);
  std::memcpy(out, v.data(), sizeof(double) * n);
}

void orc_rademacher_bits(int64_t n, uint64_t seed, int probes, uint64_t* words, int nthreads) {
  std::memset(words, 0, sizeof(uint64_t) * n);
  std::vector<std::vector<uint8_t>> bits(probes);
  auto gen = [&](int p) {
    std::seed_seq seq{static_cast<std::uint32_t>(seed), static_cast<std::uint32_t>(seed >> 32),
                      static_cast<std::uint32_t>(static_cast<uint64_t>(p)),
                      static_cast<std::uint32_t>(static_cast<uint64_t>(p) >> 32)};
    std::mt19937_64 rng(seq);
    bits[p].assign((n + 7) / 8, 0);
    for (int64_t i = 0; i < n; ++i) {
      if (rng() & 1) bits[p][i >> 3] |= static_cast<uint8_t>(1u << (i & 7));
    }
  };
  if (nthreads < 1) nthreads = 1;
  for (int p0 = 0; p0 < probes; p0 += nthreads) {
    std::vector<std::thread> th;
    for (int p = p0; p < std::min(probes, p0 + nthreads); ++p) th.emplace_back(gen, p);
    for (auto& h : th) h.join();
  }
  for (int p = 0; p < probes; ++p) {
    for (int64_t i = 0; i < n; ++i) {
      if (bits[p][i >> 3] >> (i & 7) & 1) words[i] |= (1ull << p);
    }
  }
}

int orc_wt_apply(int d, const double* gmin, const double* gmax, const int64_t* gsize,
                 int scheme, const double* x, int64_t n, const double* u, double* out) {
  return guard([&] {
    const Grid g(d, gmin, gmax, gsize);
    const Vec uu(u, u + n);
    const Vec r = wt_apply(g, scheme, x, n, uu);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}

int orc_factorized_lanczos_fused(const orc_kg* kg, const orc_stats* st, const double* kgwt_z0,
                                 const double* wt_z0, double z0_sq, double sigma_sq, int k,
                                 double* alpha, double* beta, double* dvec, double* basis,
                                 int* order) {
  return guard([&] {
    const int64_t m = kg->t->grid.m;
    const Vec a(kgwt_z0, kgwt_z0 + m), b(wt_z0, wt_z0 + m);
    const Tridiag t =
        factorized_lanczos_fused(*kg->t, st->s, a, b, z0_sq, sigma_sq, k, basis != nullptr);
    *order = static_cast<int>(t.alpha.size());
    std::memcpy(alpha, t.alpha.data(), sizeof(double) * t.alpha.size());
    if (!t.beta.empty()) std::memcpy(beta, t.beta.data(), sizeof(double) * t.beta.size());
    if (dvec) std::memcpy(dvec, t.d.data(), sizeof(double) * t.d.size());
    if (basis) {
      for (std::size_t j = 0; j < t.basis.size(); ++j) {
        std::memcpy(basis + j * m, t.basis[j].data(), sizeof(double) * m);
      }
    }
  });
}

int orc_quadrature_logdet(const double* alpha, const double* beta, int k, double probe_sq,
                          double quad_tol, double* value, int* depth) {
  return guard([&] {
    const Vec a(alpha, alpha + k), b(beta, beta + (k > 1 ? k - 1 : 0));
    const auto q = quadrature_logdet(a, b, probe_sq, quad_tol);
    *value = q.first;
    *depth = q.second;
  });
}

int orc_tridiag_eig(int k, const double* alpha, const double* beta, double* evals,
                    double* first_row) {
  return guard([&] {
    Vec lam, z;
    tridiag_eig(k, alpha, beta, lam, z);
    std::memcpy(evals, lam.data(), sizeof(double) * k);
    std::memcpy(first_row, z.data(), sizeof(double) * k);
  });
}

int orc_slq_logdet_ski_factorized(const orc_kg* kg, const orc_stats* st, int d,
                                  const double* gmin, const double* gmax, const int64_t* gsize,
                                  int scheme, const double* x, int64_t n, double sigma,
                                  int num_probes, int max_depth, double quad_tol, uint64_t seed,
                                  double* logdet, int* max_depth_used) {
  return guard([&] {
    const Grid g(d, gmin, gmax, gsize);
    const auto r = slq_logdet_ski_factorized(*kg->t, st->s, g, scheme, x, n, sigma, num_probes,
                                             max_depth, quad_tol, seed);
    *logdet = r.first;
    *max_depth_used = r.second;
  });
}

int orc_log_likelihood_gsgp(const orc_stats* st, const orc_kg* kgh, double sigma,
                            double solve_tol, int probes, int max_depth, double quad_tol,
                            uint64_t seed, int route, int64_t dense_cap, int maxiter, int d,
                            const double* gmin, const double* gmax, const int64_t* gsize,
                            int scheme, const double* x, int64_t npts, double* out, int* iout) {
  return guard([&] {
    const Toeplitz& kg = *kgh->t;
    const Stats& stats = st->s;
    const int64_t m = kg.grid.m;
    const double n = static_cast<double>(stats.n);
    const double sigma_sq = sigma * sigma;
    Vec rhat0 = kg.apply(stats.wty);
    for (auto& v : rhat0) v = -v / sigma_sq;
    const double eps_abs = solve_tol * solve_tol * stats.yty;
    const GridSolveResult solve =
        factorized_cg_grid_rhs(kg, stats, rhat0, sigma, eps_abs, -1.0, maxiter);
    if (!solve.converged) {
      throw SolverNonConvergence("log_likelihood_gsgp: mean solve did not converge",
                                 solve.residual_sq, solve.iterations);
    }
    Vec wtz(m);
    for (int64_t i = 0; i < m; ++i) wtz[i] = solve.xhat_d[i] + stats.wty[i] / sigma_sq;
    const Vec zbar = kg.apply(wtz);
    const double quad = (stats.yty - dot(stats.wty, zbar)) / sigma_sq;
    int r = route;
    if (r == 0) {
      if (x != nullptr) {
        r = 2;
      } else if (estimate_grid_kernel_condition(kg) > 1e8 && m <= dense_cap) {
        r = 3;
      } else {
        r = 1;
      }
    }
    double logdet = 0.0;
    int probes_used = 0;
    if (r == 2) {
      if (x == nullptr) {
        throw std::invalid_argument(
            "log_likelihood_gsgp: the SkiOperator logdet route needs the interpolation matrix");
      }
      const Grid g(d, gmin, gmax, gsize);
      const auto s = slq_logdet_ski_factorized(kg, stats, g, scheme, x, npts, sigma, probes,
                                               max_depth, quad_tol, seed);
      logdet = s.first - (n - static_cast<double>(m)) * std::log(sigma_sq);
      probes_used = probes;
    } else if (r == 1) {
      auto sym = [&](const Vec& u) {
        const Vec ku = kg.apply(u);
        Vec o = kg.apply(stats.apply_wtw(ku));
        for (int64_t i = 0; i < m; ++i) o[i] += sigma_sq * ku[i];
        return o;
      };
      auto kop = [&](const Vec& u) { return kg.apply(u); };
      const double s1 = slq_logdet(sym, m, probes, max_depth, 0.0, seed);
      const double s2 = slq_logdet(kop, m, probes, max_depth, 0.0, seed);
      logdet = s1 - s2;
      probes_used = 2 * probes;
    } else if (r == 3) {
      if (m > dense_cap) {
        throw std::invalid_argument(
            "log_likelihood_gsgp: grid too large for the dense logdet route");
      }
      logdet = dense_logdet_grid_system(kg, stats, sigma_sq);
    }
    const double cst = n * kLog2Pi + (n - static_cast<double>(m)) * std::log(sigma_sq);
    out[0] = -0.5 * (logdet + quad + cst);
    out[1] = logdet;
    out[2] = quad;
    out[3] = cst;
    iout[0] = probes_used;
    iout[1] = solve.iterations;
    iout[2] = r;
  });
}


int orc_posterior_cov_exact(const orc_kg* kg, const orc_stats* st, int scheme, double sigma, const double* pts,
                            int64_t ns, double tol, int maxiter, double* cov, double* max_asym, int* total_iters) {
  return guard([&] {
    const CovOut c = posterior_cov_exact(*kg->t, st->s, scheme, sigma, pts, ns, tol, maxiter);
    std::memcpy(cov, c.cov.data(), sizeof(double) * ns * ns);
    *max_asym = c.max_asymmetry;
    *total_iters = c.total_iterations;
  });
}

// low-rank covariance: rank used, then the cov matrix at ns points and (optionally) one query
int orc_posterior_cov_lowrank(const orc_kg* kg, const orc_stats* st, int scheme, double sigma, int64_t rank,
                              const double* pts, int64_t ns, double* cov, const double* qx, const double* qx2,
                              double* qout, int* rank_used) {
  return guard([&] {
    const LowRank lr = posterior_cov_lowrank(*kg->t, st->s, sigma, rank);
    *rank_used = lr.k;
    if (ns > 0) {
      const Vec c = lowrank_cov_matrix(*kg->t, lr, scheme, pts, ns);
      std::memcpy(cov, c.data(), sizeof(double) * ns * ns);
    }
    if (qx && qx2 && qout) *qout = lowrank_query(*kg->t, lr, scheme, qx, qx2);
  });
}

}  // extern "C"
