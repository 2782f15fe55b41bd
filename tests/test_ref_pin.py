"""Pins the oracle restatement (oracle/gsgp_oracle.cpp) against the REFERENCE'S OWN SOURCES.

``oracle.ref`` is the same front-end bound to ``oracle/_ref/libgsgp_ref.so``: the unmodified
/root/reference/proj sources (kernels, grid, interp, solvers, gp .cpp) compiled where they lie
against self-written stand-ins for the absent Eigen3 / FFTW3 / json headers
(oracle/refshim/README.md).  The reference's control flow and arithmetic are therefore its
own; only the containers and the dense-algebra primitives (dot products, the FFT) are the
stand-ins'.  Bounds: bit-exact wherever the order of operations is fixed by the reference's
own loops (grids, stencils, weights, the hash-map accumulation, CSR structure, probes,
next_fast_fft_size, generator); round-off level where a reduction or the FFT is involved.

CPU only; skipped when the reference library is neither built nor buildable.
"""
import numpy as np
import pytest

import oracle as O
import oracle.ref as R

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref/libgsgp_ref.so not built (needs /root/reference)")

CASES = [(1, [40]), (2, [20, 17]), (3, [12, 9, 8])]


def _grids(d, sizes, scheme=O.CUBIC):
    lo, hi = [0.0] * d, [1.0] * d
    return O.fit_grid_to_data(lo, hi, sizes, scheme), R.fit_grid_to_data(lo, hi, sizes, scheme)


def _rows(d, sizes, n, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.random((n, d))
    y = rng.standard_normal(n)
    k = min(64, n // 4)
    # rows on grid nodes, inside the 1e-9 snap band, and on the upper data bound
    x[:k] = np.round(x[:k] * (np.array(sizes) - 5)) / (np.array(sizes) - 5)
    x[k:2 * k] = x[:k] + rng.uniform(-2e-11, 2e-11, (k, d))
    x[2 * k] = 1.0
    x[2 * k + 1] = 0.0
    return np.clip(x, 0.0, 1.0), y


def test_reference_library_identifies_itself():
    assert "interp.cpp" in R.ref_build_info()


@pytest.mark.parametrize("scheme", [O.LINEAR, O.CUBIC])
@pytest.mark.parametrize("d,sizes", CASES)
def test_grid_and_weights_bit_exact(d, sizes, scheme):
    g, gr = _grids(d, sizes, scheme)
    assert list(g.mins) == list(gr.mins) and list(g.maxs) == list(gr.maxs)
    x, _ = _rows(d, sizes, 600)
    for i in range(x.shape[0]):
        a, b = O.interp_weights(g, x[i], scheme), R.interp_weights(gr, x[i], scheme)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("scheme", [O.LINEAR, O.CUBIC])
def test_fit_grid_errors(scheme):
    for mod in (O, R):
        with pytest.raises(mod.OracleError) as e:
            mod.fit_grid_to_data([0.0], [1.0], [3], scheme)
        assert "need at least" in str(e.value)
        with pytest.raises(mod.OracleError) as e:
            mod.fit_grid_to_data([1.0], [1.0], [16], scheme)
        assert "empty data range" in str(e.value)


@pytest.mark.parametrize("scheme", [O.LINEAR, O.CUBIC])
@pytest.mark.parametrize("d,sizes", CASES)
def test_sufficient_stats_bit_exact(d, sizes, scheme):
    """One pass in stream order: the restatement's statistics equal the reference's bit for bit
    (same hash-map accumulation order, same setFromTriplets structure)."""
    g, gr = _grids(d, sizes, scheme)
    x, y = _rows(d, sizes, 6000, seed=d)
    so, sr = O.sufficient_stats(g, x, y, scheme), R.sufficient_stats(gr, x, y, scheme)
    for a, b in zip(so.csr(), sr.csr()):
        assert np.array_equal(a, b)
    assert so.yty == sr.yty and so.n == sr.n == 6000
    assert so.max_row_nnz() == sr.max_row_nnz()
    v = np.random.default_rng(1).standard_normal(g.m)
    assert np.array_equal(so.apply_wtw(v), sr.apply_wtw(v))
    # fp32 rows (configs 2-4) widen the same way
    x32, y32 = x.astype(np.float32), y.astype(np.float32)
    s32, r32 = O.sufficient_stats(g, x32, y32, scheme), R.sufficient_stats(gr, x32, y32, scheme)
    for a, b in zip(s32.csr(), r32.csr()):
        assert np.array_equal(a, b)


def test_merge_of_shards():
    """Shards combined with the reference's merge() (interp.cpp:202-210): same structure, values
    to round-off (the restatement merges as a tree, the reference binding in shard order)."""
    g, gr = _grids(2, [20, 17])
    x, y = _rows(2, [20, 17], 20000, seed=5)
    one = R.sufficient_stats(gr, x, y)
    so, sr = O.sufficient_stats(g, x, y, nthreads=4), R.sufficient_stats(gr, x, y, nthreads=4)
    co, cr, c1 = so.csr(), sr.csr(), one.csr()
    assert np.array_equal(co[0], cr[0]) and np.array_equal(co[1], cr[1])
    assert np.array_equal(c1[0], cr[0]) and np.array_equal(c1[1], cr[1])
    scale = np.abs(c1[2]).max()
    assert np.abs(co[2] - cr[2]).max() <= 1e-13 * scale
    assert np.abs(c1[2] - cr[2]).max() <= 1e-12 * scale
    assert so.n == sr.n == one.n and abs(sr.yty - one.yty) <= 1e-12 * one.yty


@pytest.mark.parametrize("scheme", [O.LINEAR, O.CUBIC])
def test_out_of_grid_rows_report_the_same_row_and_text(scheme):
    g, gr = _grids(2, [12, 12], scheme)
    x, y = _rows(2, [12, 12], 500)
    for bad, val in ((137, 1.7), (9, -0.4)):
        xb = x.copy()
        xb[bad, 1] = val
        errs = []
        for mod, grid in ((O, g), (R, gr)):
            with pytest.raises(mod.OracleError) as e:
                mod.sufficient_stats(grid, xb, y, scheme)
            errs.append((e.value.code, e.value.row, str(e.value)))
        assert errs[0] == errs[1]
        assert errs[0][0] == O.OUT_OF_GRID and errs[0][1] == bad + 1
    # a point inside the grid whose cubic stencil leaves it (grid not fit to the data)
    tight_o, tight_r = O.Grid([0.0, 0.0], [1.0, 1.0], [12, 12]), R.Grid([0.0, 0.0], [1.0, 1.0], [12, 12])
    if scheme == O.CUBIC:
        errs = []
        for mod, grid in ((O, tight_o), (R, tight_r)):
            with pytest.raises(mod.OracleError) as e:
                mod.interp_weights(grid, [0.01, 0.5], scheme)
            errs.append((e.value.code, str(e.value)))
        assert errs[0] == errs[1] and "stencil leaves the grid" in errs[0][1]


@pytest.mark.parametrize("d,sizes", CASES + [(1, [97]), (2, [33, 50])])
def test_toeplitz_operator(d, sizes):
    g, gr = _grids(d, sizes)
    ls = [0.31, 0.2, 0.45][:d]
    ko, kr = O.ToeplitzOperator(g, ls, 1.5, 0.1), R.ToeplitzOperator(gr, ls, 1.5, 0.1)
    assert list(ko.embed_shape()) == list(kr.embed_shape())
    assert np.array_equal(ko.generator(), kr.generator())
    v = np.random.default_rng(2).standard_normal(g.m)
    a, b = ko.apply(v), kr.apply(v)
    assert np.abs(a - b).max() <= 1e-12 * np.abs(a).max()  # two FFT implementations
    if g.m <= 400:
        assert np.array_equal(ko.dense(), kr.dense())
        assert np.abs(kr.dense() @ v - b).max() <= 1e-11 * np.abs(b).max()


def test_next_fast_fft_size():
    for x in list(range(0, 300)) + [1023, 1025, 4097, 19999, 65537]:
        assert O.next_fast_fft_size(x) == R.next_fast_fft_size(x)


def _problem(d, sizes, n=8000, seed=3, sigma=0.1):
    g, gr = _grids(d, sizes)
    x, y = _rows(d, sizes, n, seed=seed)
    y = np.sin(4.0 * x.sum(axis=1)) + sigma * y
    # lengthscales of ~1.3 grid spacings keep K_G well conditioned, so the CG / Lanczos recurrences
    # stay comparable term by term (on ill-conditioned K_G any two roundings part after ~10 steps)
    ls = [1.3 / (s - 5) for s in sizes]
    so, sr = O.sufficient_stats(g, x, y), R.sufficient_stats(gr, x, y)
    ko, kr = O.ToeplitzOperator(g, ls, 1.2, sigma), R.ToeplitzOperator(gr, ls, 1.2, sigma)
    return g, gr, x, y, so, sr, ko, kr, sigma


@pytest.mark.parametrize("d,sizes", CASES)
def test_factorized_cg_grid_rhs(d, sizes):
    g, gr, x, y, so, sr, ko, kr, sigma = _problem(d, sizes)
    r0 = -ko.apply(so.wty) / sigma ** 2
    a = O.factorized_cg_grid_rhs(ko, so, r0, sigma, rel_tol=1e-6, maxiter=800)
    b = R.factorized_cg_grid_rhs(kr, sr, r0, sigma, rel_tol=1e-6, maxiter=800)
    assert a.converged and b.converged
    k = min(10, a.iterations, b.iterations)
    assert np.abs(a.alphas[:k] / b.alphas[:k] - 1).max() <= 1e-8
    assert np.abs(a.betas[:k - 1] / b.betas[:k - 1] - 1).max() <= 1e-8
    assert np.abs(a.residual_trace[:k] / b.residual_trace[:k] - 1).max() <= 1e-8
    assert abs(a.iterations - b.iterations) <= max(2, a.iterations // 50)
    assert np.abs(a.xhat_d - b.xhat_d).max() <= 2e-5 * np.abs(b.xhat_d).max()
    # absolute tolerance form and the maxiter exit
    c = O.factorized_cg_grid_rhs(ko, so, r0, sigma, eps_abs=1e-12 * a.residual_trace[0], maxiter=3)
    e = R.factorized_cg_grid_rhs(kr, sr, r0, sigma, eps_abs=1e-12 * a.residual_trace[0], maxiter=3)
    assert c.iterations == e.iterations == 3 and not c.converged and not e.converged
    assert c.residual_sq == pytest.approx(e.residual_sq, rel=1e-10)
    assert np.abs(c.xhat_d - e.xhat_d).max() <= 1e-10 * np.abs(e.xhat_d).max()


@pytest.mark.parametrize("d,sizes", CASES)
def test_posterior_mean_and_prediction(d, sizes):
    g, gr, x, y, so, sr, ko, kr, sigma = _problem(d, sizes)
    ma, ia, _ = O.posterior_mean_gsgp(ko, so, sigma, 1e-7, 3000)
    mb, ib, _ = R.posterior_mean_gsgp(kr, sr, sigma, 1e-7, 3000)
    assert abs(ia - ib) <= max(3, ib // 20)
    assert np.abs(ma - mb).max() <= 1e-5 * np.abs(mb).max()
    pts = np.random.default_rng(4).random((200, d))
    pa, pb = O.predict_mean(g, mb, pts), R.predict_mean(gr, mb, pts)
    assert np.abs(pa - pb).max() <= 1e-14 * np.abs(pb).max()
    with pytest.raises(R.OracleError) as e:
        R.posterior_mean_gsgp(kr, sr, sigma, 1e-12, 2)
    assert e.value.code == O.NONCONVERGENCE
    with pytest.raises(O.OracleError) as e2:
        O.posterior_mean_gsgp(ko, so, sigma, 1e-12, 2)
    assert e2.value.code == O.NONCONVERGENCE and str(e.value) == str(e2.value)


def test_probes_bit_exact():
    for seed, p in ((0, 0), (7, 3), (2 ** 40 + 5, 29), (123456789, 2 ** 33)):
        assert np.array_equal(O.rademacher_probe(4096, seed, p), R.rademacher_probe(4096, seed, p))
    assert np.array_equal(O.rademacher_bits(3000, 11, 30), R.rademacher_bits(3000, 11, 30))


@pytest.mark.parametrize("d,sizes", CASES)
def test_lanczos_and_quadrature(d, sizes):
    g, gr, x, y, so, sr, ko, kr, sigma = _problem(d, sizes, n=3000)
    v = O.rademacher_probe(x.shape[0], 5, 1)
    wt = O.wt_apply(g, x, v)
    wtr = R.wt_apply(gr, x, v)
    assert np.abs(wt - wtr).max() <= 1e-13 * np.abs(wtr).max()
    kg = kr.apply(wtr)
    k = 20
    a = O.factorized_lanczos_fused(ko, so, kg, wtr, float(v @ v), sigma ** 2, k)
    b = R.factorized_lanczos_fused(kr, sr, kg, wtr, float(v @ v), sigma ** 2, k)
    assert len(a["alpha"]) == len(b["alpha"])
    assert np.abs(a["alpha"] / b["alpha"] - 1).max() <= 1e-7 and np.abs(a["beta"] / b["beta"] - 1).max() <= 1e-7
    assert np.abs(a["d"] - b["d"]).max() <= 1e-7 * max(np.abs(b["d"]).max(), 1e-300)
    for tol in (0.0, 0.01):
        qa = O.quadrature_logdet(b["alpha"], b["beta"], float(v @ v), tol)
        qb = R.quadrature_logdet(b["alpha"], b["beta"], float(v @ v), tol)
        assert qa[1] == qb[1] and abs(qa[0] - qb[0]) <= 1e-9 * abs(qb[0])


@pytest.mark.parametrize("route", ["ski-operator", "symmetric-grid", "dense", "auto"])
def test_log_likelihood_routes(route):
    d, sizes = 2, [14, 12]
    g, gr, x, y, so, sr, ko, kr, sigma = _problem(d, sizes, n=2500)
    kw = dict(solve_tol=1e-9, probes=6, max_depth=40, quad_tol=0.0, seed=3, route=route, maxiter=4000)
    with_w = route in ("ski-operator", "auto")
    a = O.log_likelihood_gsgp(so, ko, sigma, grid=g, x=x if with_w else None, **kw)
    b = R.log_likelihood_gsgp(sr, kr, sigma, grid=gr, x=x if with_w else None, **kw)
    assert a["logdet_route"] == b["logdet_route"] and a["probes_used"] == b["probes_used"]
    assert abs(a["quad_term"] - b["quad_term"]) <= 1e-6 * abs(b["quad_term"])
    assert a["const_term"] == b["const_term"]
    # the paired symmetric-grid estimate subtracts two large SLQ sums: looser bound
    tol = 1e-4 if b["logdet_route"] == "symmetric-grid-slq" else 1e-6
    assert abs(a["logdet_term"] - b["logdet_term"]) <= tol * max(abs(b["logdet_term"]), 1.0)
    assert abs(a["loglik"] - b["loglik"]) <= tol * abs(b["loglik"])


def test_auto_route_without_w_follows_the_condition_estimate():
    d, sizes = 2, [14, 12]
    g, gr, x, y, so, sr, ko, kr, sigma = _problem(d, sizes, n=2500)
    a = O.log_likelihood_gsgp(so, ko, sigma, solve_tol=1e-9, probes=4, max_depth=30, quad_tol=0.0, maxiter=4000)
    b = R.log_likelihood_gsgp(sr, kr, sigma, solve_tol=1e-9, probes=4, max_depth=30, quad_tol=0.0, maxiter=4000)
    assert a["logdet_route"] == b["logdet_route"]


def test_posterior_covariance():
    d, sizes = 2, [14, 12]
    g, gr, x, y, so, sr, ko, kr, sigma = _problem(d, sizes, n=2500)
    pts = np.random.default_rng(6).random((5, d))
    ca, cb = O.posterior_cov_exact(ko, so, sigma, pts), R.posterior_cov_exact(kr, sr, sigma, pts)
    # cov = prior − correction cancels to ~4e-4 of the prior scale (outputscale 1.2)
    assert np.abs(ca["cov"] - cb["cov"]).max() <= 1e-7 * 1.2
    assert ca["total_iterations"] > 0 and abs(ca["total_iterations"] - cb["total_iterations"]) <= 5 * len(pts)
    la = O.posterior_cov_lowrank(ko, so, sigma, 12, points=pts, query=(pts[0], pts[1]))
    lb = R.posterior_cov_lowrank(kr, sr, sigma, 12, points=pts, query=(pts[0], pts[1]))
    assert la["rank"] == lb["rank"]
    assert np.abs(la["cov"] - lb["cov"]).max() <= 1e-7 * 1.2
    assert abs(la["query"] - lb["query"]) <= 1e-7 * 1.2
