// C++ host-API test: the gsgp_b200:: mirror of the reference API (include/gsgp_b200.hpp)
// driving libgsgpc.so, checked against the CPU oracle (test infrastructure).
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "gsgp_b200.hpp"
#include "gsgp_oracle.h"

using namespace gsgp_b200;

static int failures = 0;
#define CHECK(cond, what)                                              \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, what); \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

struct MemoryRowStream : RowStream {  // io.hpp:49-60
  const std::vector<double>& x;
  const std::vector<double>& y;
  int d;
  size_t pos = 0;
  MemoryRowStream(const std::vector<double>& x_, const std::vector<double>& y_, int d_) : x(x_), y(y_), d(d_) {}
  int dim() const override { return d; }
  bool next(std::vector<double>& xr, double& yr) override {
    if (pos >= y.size()) return false;
    xr.assign(x.begin() + pos * d, x.begin() + (pos + 1) * d);
    yr = y[pos++];
    return true;
  }
};

static double lcg(uint64_t& s) {
  s = s * 6364136223846793005ull + 1442695040888963407ull;
  return static_cast<double>(s >> 11) / 9007199254740992.0;
}

static double max_rel(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0.0, den = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    num = std::max(num, std::fabs(a[i] - b[i]));
    den = std::max(den, std::fabs(b[i]));
  }
  return den > 0 ? num / den : num;
}

int main() {
  const int d = 2;
  const int64_t n = 50000;
  std::vector<double> x(n * d), y(n);
  uint64_t s = 42;
  for (int64_t i = 0; i < n; ++i) {
    x[i * d] = lcg(s);
    x[i * d + 1] = lcg(s);
    y[i] = std::sin(6.0 * x[i * d]) * std::cos(4.0 * x[i * d + 1]) + 0.05 * (lcg(s) - 0.5);
  }
  const Grid grid = fit_grid_to_data({0.0, 0.0}, {1.0, 1.0}, {40, 36}, InterpScheme::Cubic);
  MemoryRowStream stream(x, y, d);
  auto stats = std::make_shared<SufficientStats>(sufficient_stats(grid, InterpScheme::Cubic, stream));
  CHECK(stats->n() == n, "n");

  // oracle
  double gmin[2] = {grid.min(0), grid.min(1)}, gmax[2] = {grid.max(0), grid.max(1)};
  int64_t gsz[2] = {grid.size(0), grid.size(1)};
  orc_stats* os = nullptr;
  CHECK(orc_sufficient_stats(d, gmin, gmax, gsz, 1, x.data(), y.data(), n, 4, &os) == ORC_OK, "oracle stats");
  int64_t om, on, onnz;
  double oyty;
  orc_stats_info(os, &om, &on, &onnz, &oyty);
  std::vector<int64_t> rp(om + 1), col(onnz);
  std::vector<double> val(onnz), owty(om);
  orc_stats_export(os, rp.data(), col.data(), val.data(), owty.data());
  CHECK(max_rel(stats->wty(), owty) <= 1e-10, "wty");
  CHECK(std::fabs(stats->yty() - oyty) <= 1e-12 * oyty, "yty");
  const auto csr = stats->wtw();
  CHECK(csr.row_ptr == rp && csr.col == col, "wtw structure");
  CHECK(max_rel(csr.val, val) <= 1e-10, "wtw values");
  CHECK(stats->max_row_nnz() == orc_stats_max_row_nnz(os) && stats->max_row_nnz() <= 49, "Claim 2 nnz");

  // K_G and posterior mean
  const KernelSpec spec(Hyperparams(0.5, {0.08, 0.1}, 1.0));
  auto kg = std::make_shared<ToeplitzOperator>(grid, spec);
  orc_kg* okg = nullptr;
  double ls[2] = {0.08, 0.1};
  CHECK(orc_kg_create(d, gmin, gmax, gsz, ls, 1.0, 0.5, &okg) == ORC_OK, "oracle kg");
  std::vector<double> v(om);
  for (auto& e : v) e = lcg(s) - 0.5;
  std::vector<double> okv(om);
  orc_kg_apply(okg, v.data(), okv.data());
  CHECK(max_rel(kg->apply(v), okv) <= 1e-10, "K_G v");
  const PosteriorModel model = posterior_mean_gsgp(stats, kg, spec, InterpScheme::Cubic, 0.5, 1e-8);
  std::vector<double> omc(om);
  int oit = 0;
  double ors = 0;
  CHECK(orc_posterior_mean_gsgp(okg, os, 0.5, 1e-8, 1000, omc.data(), &oit, &ors) == ORC_OK, "oracle mean");
  CHECK(max_rel(model.mean_coeffs, omc) <= 1e-5, "mean coeffs");
  // ill-conditioned enough that counts drift with the summation order
  CHECK(std::abs(model.solve_iterations - oit) <= std::max(2, oit / 10), "iterations");
  std::vector<double> tp = {0.3, 0.4, 0.71, 0.2, 0.5, 0.5};
  std::vector<double> opred(3);
  orc_predict_mean(d, gmin, gmax, gsz, 1, omc.data(), tp.data(), 3, opred.data());
  CHECK(max_rel(model.predict_mean(tp), opred) <= 1e-5, "predict");

  // errors: the reference's std::invalid_argument with the stream row
  std::vector<double> xb = {0.5, 0.5, 2.0, 0.5, 0.4, 0.4}, yb = {1, 2, 3};
  MemoryRowStream bad(xb, yb, d);
  bool threw = false;
  try {
    sufficient_stats(grid, InterpScheme::Cubic, bad);
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()).find("stream row 2") != std::string::npos;
  }
  CHECK(threw, "out-of-grid row 2");
  // SolverNonConvergence
  threw = false;
  try {
    posterior_mean_gsgp(stats, kg, spec, InterpScheme::Cubic, 0.5, 1e-14, 2);
  } catch (const SolverNonConvergence& e) {
    threw = e.iterations == 2;
  }
  CHECK(threw, "nonconvergence");

  // stats file round trip
  save_stats("/tmp/gsgp_b200_test.gsgpsst", *stats, grid, InterpScheme::Cubic);
  const StatsFile sf = load_stats("/tmp/gsgp_b200_test.gsgpsst");
  CHECK(sf.stats.n() == n && sf.stats.wtw().val == csr.val, "stats round trip");

  // several GPUs from one process: a group listing device 0 twice (one GPU per test box) —
  // the merged statistics equal the oracle's on all rows, on every device
  {
    const DeviceGroup group({0, 0});
    CHECK(group.size() == 2, "group size");
    const std::vector<SufficientStats> gs = group.sufficient_stats(grid, InterpScheme::Cubic, x, y);
    for (const SufficientStats& st : gs) {
      CHECK(st.n() == n, "group n");
      CHECK(max_rel(st.wty(), owty) <= 1e-10, "group wty");
      const auto gc = st.wtw();
      CHECK(gc.row_ptr == rp && gc.col == col, "group wtw structure");
      CHECK(max_rel(gc.val, val) <= 1e-10, "group wtw values");
    }
  }

  orc_stats_destroy(os);
  orc_kg_destroy(okg);
  if (failures == 0) std::printf("cpp api OK: iters=%d (oracle %d)\n", model.solve_iterations, oit);
  return failures == 0 ? 0 : 1;
}
