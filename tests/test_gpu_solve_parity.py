"""Solve parity on the BASELINE configurations, on IDENTICAL statistics.

The GPU and oracle solvers are fed the same W^T W, W^T y, yᵀy and n, so they differ only in
their own rounding:
  * config 1 (full n = 1e6): the ORACLE's statistics written in the reference's GSGPSST1 layout
    (io.cpp:192-221) and loaded by the library (gsgpc_stats_load);
  * configs 2 (full n = 1e7) and 3 (1e6-row prefix): the GPU's statistics exported as CSR and
    loaded by the oracle (the oracle's own hash-map precompute of 1e7 3-D rows takes minutes);
  * config 5 (1e6-row prefix): the log-likelihood against the oracle's value computed once on
    the same numpy rows (tests/golden/loglik_config5.json, tests/golden/make_loglik5_golden.py:
    ~25 min of oracle CPU time at solve_tol 1e-8).

How far two valid roundings of the reference's own arithmetic move the solve is measured in
the same tests: the oracle is run twice, with K_G applied by the restated circulant FFT
(grid.cpp:193-235) and by direct Toeplitz sums (same operator, different rounding).  On these
ill-conditioned systems the CG trajectories of the two ORACLE runs part after ~20 iterations
(config 3) and their iteration counts differ by tens (config 1: 795 vs 833); the GPU's must stay
inside that measured spread, and its leading traces must agree to round-off.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_2101_11751_b200 as G
from helpers import oracle_stats_from_gpu, rel_err, write_gsgpsst1

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def _threads():
    O.set_threads(os.cpu_count() or 8)
    yield


def ogrid(g):
    return O.Grid([g.min(k) for k in range(g.dim())], [g.max(k) for k in range(g.dim())],
                  [g.size(k) for k in range(g.dim())])


def kgs(cfg, og):
    fft = O.ToeplitzOperator(og, list(cfg.lengthscales), cfg.outputscale, cfg.noise_std)
    direct = O.ToeplitzOperator(og, list(cfg.lengthscales), cfg.outputscale, cfg.noise_std)
    direct.set_direct()
    return fft, direct


def rel_each(a, b):
    a, b = np.asarray(a), np.asarray(b)
    n = min(len(a), len(b))
    return np.abs(a[:n] - b[:n]) / np.maximum(np.abs(b[:n]), 1e-300)


def test_config1_posterior_mean_on_oracle_statistics(tmp_path):
    """BASELINE config 1 at full n: posterior_mean_gsgp (gp.cpp:326-352) at tol 1e-6 and 1e-8 on
    the oracle's statistics loaded through GSGPSST1.

    This system is numerically singular (lengthscale / spacing ≈ 24), and its CG iteration count
    is set by round-off: the oracle itself, on the same statistics, stops at different counts
    with its FFT and its direct-sum K_G, and again on the same rows accumulated with another
    thread count (another hash-map merge order).  Measured here: four oracle variants; the GPU's
    count must lie within their span (plus one), its coefficients within 1e-5 (1e-6 at tol
    1e-8) or twice the oracle variants' own spread, its predictions within 1e-5 / 1e-7."""
    from paper_2101_11751_b200 import synthetic as S

    cfg = S.CONFIGS[1]
    g = S.grid_for(cfg)
    og = ogrid(g)
    x, y = S.generate(1)
    ost = O.sufficient_stats(og, x, y, nthreads=os.cpu_count() or 8)
    ost1 = O.sufficient_stats(og, x, y, nthreads=3)  # same rows, another merge order
    rp, col, val, wty = ost.csr()
    p = str(tmp_path / "c1.gsgpsst")
    write_gsgpsst1(p, (og.mins, og.maxs, og.sizes), 1, rp, col, val, wty, ost.yty, ost.n)
    gst = G.load_stats(p).stats
    assert gst.n() == ost.n == cfg.n and gst.yty() == ost.yty
    assert np.array_equal(gst.wty(), wty)
    spec = S.kernel_for(cfg)
    kg = G.ToeplitzOperator(g, spec)
    okg, okd = kgs(cfg, og)
    tp = np.linspace(-10.0, 10.0, 1000).reshape(-1, 1)
    for tol, mean_tol, pred_tol in ((1e-6, 1e-5, 1e-5), (1e-8, 1e-6, 1e-7)):
        variants = [O.posterior_mean_gsgp(k, st, cfg.noise_std, tol, 5000) for st in (ost, ost1) for k in (okg, okd)]
        omc, oit, _ = variants[0]
        its = [v[1] for v in variants]
        spread_mean = max(rel_err(v[0], omc) for v in variants[1:])
        model = G.posterior_mean_gsgp(gst, kg, spec, G.InterpScheme.Cubic, cfg.noise_std, tol, 5000)
        assert min(its) - 1 <= model.solve_iterations <= max(its) + 1, (tol, model.solve_iterations, its)
        assert rel_err(model.mean_coeffs, omc) <= max(mean_tol, 2 * spread_mean), (tol, spread_mean)
        assert rel_err(model.predict_mean(tp), O.predict_mean(og, omc, tp)) <= pred_tol, tol
    # the leading CG traces agree to round-off (solvers.cpp:271-336)
    r0 = -okg.apply(wty) / cfg.noise_variance
    ores = O.factorized_cg_grid_rhs(okg, ost, r0, cfg.noise_std, eps_abs=1e-30, maxiter=20)
    gres = G.factorized_cg_grid_rhs(kg, gst, r0, cfg.noise_std, G.GridRhsTolerance(eps_abs=1e-30), 20)
    assert rel_each(gres.alphas, ores.alphas).max() <= 1e-10
    assert rel_each(gres.betas, ores.betas).max() <= 1e-10
    assert rel_each(gres.residual_trace, ores.residual_trace).max() <= 1e-10


@pytest.mark.parametrize("cid,n,lead,loose_at", [(2, None, 20, 50), (3, 1_000_000, 16, None)])
def test_cg_traces_on_identical_statistics(cid, n, lead, loose_at):
    """factorized_cg_grid_rhs on the posterior-mean system of configs 2 (full n) and 3 (1e6-row
    prefix): α, β, ρ per iteration against the oracle over a fixed window.  The first `lead`
    iterations agree to 1e-10; later the oracle's own FFT and direct-K_G runs part as well
    (config 3: by ~1e-2 at iteration 24), so the GPU's deviation is bounded there by that
    measured sensitivity."""
    from paper_2101_11751_b200 import synthetic as S

    cfg = S.CONFIGS[cid]
    g = S.grid_for(cfg)
    og = ogrid(g)
    x, y = S.generate(cid, n)
    gst = G.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
    ost = oracle_stats_from_gpu(gst)
    kg = G.ToeplitzOperator(g, S.kernel_for(cfg))
    okg, okd = kgs(cfg, og)
    wty = gst.wty()
    assert rel_err(kg.apply(wty), okg.apply(wty)) <= 1e-12
    r0 = -okg.apply(wty) / cfg.noise_variance
    it = max(lead, loose_at or 0)
    ores = O.factorized_cg_grid_rhs(okg, ost, r0, cfg.noise_std, eps_abs=1e-30, maxiter=it)
    dres = O.factorized_cg_grid_rhs(okd, ost, r0, cfg.noise_std, eps_abs=1e-30, maxiter=it)
    gres = G.factorized_cg_grid_rhs(kg, gst, r0, cfg.noise_std, G.GridRhsTolerance(eps_abs=1e-30), it)
    assert gres.iterations == ores.iterations == it
    for name in ("alphas", "betas", "residual_trace"):
        a = rel_each(getattr(gres, name)[:lead], getattr(ores, name)[:lead])
        assert a.max() <= 1e-10, (name, a.max())
    if loose_at:
        gd = rel_each(gres.alphas[:loose_at], ores.alphas[:loose_at]).max()
        dd = rel_each(dres.alphas[:loose_at], ores.alphas[:loose_at]).max()
        assert gd <= max(1e-6, 100 * dd), (gd, dd)


def test_config5_loglik_matches_oracle_golden():
    """log_likelihood_gsgp (gp.cpp:158-240), SkiOperator route: 30 probes of the reference's
    generator, depth 50, quad_tol 0, solve_tol 1e-8, on a 1e6-row prefix of BASELINE config 5
    (numpy rows, identical on every machine) — loglik, logdet and quadratic terms within 1e-5 of
    the oracle (tests/golden/loglik_config5.json)."""
    from paper_2101_11751_b200 import synthetic as S

    path = os.path.join(GOLD, "loglik_config5.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/loglik_config5.json not generated")
    gold = json.load(open(path))
    cfg = S.CONFIGS[5]
    g = S.grid_for(cfg)
    x, y = S.generate(5, gold["n"])
    acc = G.SufficientStatsAccumulator(g)
    acc.enable_probes(gold["options"]["probes"], seed=gold["options"]["seed"])
    acc.add(x, y)
    st = acc.finalize()
    chk = gold["stats_check"]
    assert st.n() == chk["n"]
    assert abs(st.yty() - chk["yty"]) <= 1e-12 * chk["yty"]
    assert abs(st.wty().sum() - chk["wty_sum"]) <= 1e-10 * chk["wty_abs_sum"]
    o = gold["options"]
    kg = G.ToeplitzOperator(g, S.kernel_for(cfg))
    opts = G.LoglikOptions(solve_tol=o["solve_tol"], probes=o["probes"], slq=G.SlqOptions(o["max_depth"], o["quad_tol"]),
                           seed=o["seed"], maxiter=o["maxiter"], route=G.LogdetRoute.SkiOperator)
    r = G.log_likelihood_gsgp(st, kg, cfg.noise_std, opts)
    ref = gold["oracle"]
    assert r.const_term == pytest.approx(ref["const_term"], rel=1e-14)
    for mine, key in ((r.loglik, "loglik"), (r.logdet_term, "logdet_term"), (r.quad_term, "quad_term")):
        assert abs(mine - ref[key]) <= 1e-5 * abs(ref[key]), (key, mine, ref[key])
    assert r.probes_used == ref["probes_used"] == 30
