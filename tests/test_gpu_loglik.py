"""GPU parity of the probe images, probe-batched EFLA and the log-likelihood on every
LogdetRoute (SkiOperator, SymmetricGrid, Dense, Auto) against the oracle on identical probes
(same reference generator)."""
import numpy as np
import pytest

import oracle as O
import paper_2101_11751_b200 as G
from helpers import rel_err

pytestmark = pytest.mark.gpu


def ogrid(g):
    return O.Grid([g.min(k) for k in range(g.dim())], [g.max(k) for k in range(g.dim())],
                  [g.size(k) for k in range(g.dim())])


def make_case(d=3, sizes=(10, 9, 8), n=6000, seed=5):
    rng = np.random.default_rng(seed)
    x = rng.random((n, d))
    om = rng.standard_normal((20, d)) / 0.3
    y = np.cos(x @ om.T).sum(axis=1) / 5.0 + 0.1 * rng.standard_normal(n)
    g = G.fit_grid_to_data(np.zeros(d), np.ones(d), sizes)
    return g, x, y


@pytest.mark.parametrize("d,sizes,n", [(1, (40,), 5000), (2, (16, 14), 5000), (3, (10, 9, 8), 5000),
                                       (2, (600, 600), 150_000)])  # 512-cell buckets: staged slice scatter
def test_probe_images_match_oracle(d, sizes, n):
    g, x, y = make_case(d, sizes, n=n)
    acc = G.SufficientStatsAccumulator(g)
    acc.enable_probes(5, seed=7)
    acc.add(x[:2000], y[:2000])  # streams continue across batches
    acc.add(x[2000:], y[2000:])
    ost = O.sufficient_stats(ogrid(g), x, y, nthreads=8) if n > 10000 else None
    if ost is not None:  # the rows' statistics on the same (staged) path
        assert rel_err(acc.finalize().wty(), ost.csr()[3]) <= 1e-10
    st = acc.finalize()
    img = st.probe_images()
    og = ogrid(g)
    for p in range(5):
        v = O.rademacher_probe(x.shape[0], 7, p)
        ref = O.wt_apply(og, x, v)
        assert rel_err(img[p], ref) <= 1e-10, p


def test_efla_matches_oracle():
    g, x, y = make_case()
    sigma = 0.1
    spec = G.KernelSpec(G.Hyperparams(sigma, [0.2, 0.25, 0.3], 1.0))
    st = G.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
    og = ogrid(g)
    ost = O.sufficient_stats(og, x, y)
    okg = O.ToeplitzOperator(og, [0.2, 0.25, 0.3], 1.0, sigma)
    kg = G.ToeplitzOperator(g, spec)
    P, k = 3, 25
    wts, kwts, z = [], [], []
    for p in range(P):
        v = O.rademacher_probe(x.shape[0], 0, p)
        w = O.wt_apply(og, x, v)
        wts.append(w)
        kwts.append(okg.apply(w))
        z.append(float(v @ v))
    a, b, order = G.factorized_lanczos_fused(kg, st, np.array(kwts), np.array(wts), np.array(z), sigma * sigma, k)
    for p in range(P):
        ref = O.factorized_lanczos_fused(okg, ost, kwts[p], wts[p], z[p], sigma * sigma, k)
        assert order[p] == len(ref["alpha"])
        o = order[p]
        assert rel_err(a[p, :o], ref["alpha"]) <= 1e-6
        assert rel_err(b[p, : o - 1], ref["beta"]) <= 1e-6


def test_loglik_matches_oracle():
    g, x, y = make_case(n=8000)
    sigma = 0.1
    ls = [0.2, 0.25, 0.3]
    spec = G.KernelSpec(G.Hyperparams(sigma, ls, 1.0))
    acc = G.SufficientStatsAccumulator(g)
    acc.enable_probes(30, seed=0)
    acc.add(x, y)
    st = acc.finalize()
    kg = G.ToeplitzOperator(g, spec)
    # data-fit solve to 1e-9 so the quadratic terms of the two sides agree far below 1e-5
    opts = G.LoglikOptions(solve_tol=1e-9, probes=30, slq=G.SlqOptions(max_depth=50, quad_tol=0.0), seed=0,
                           maxiter=5000)
    r = G.log_likelihood_gsgp(st, kg, sigma, opts)
    og = ogrid(g)
    ost = O.sufficient_stats(og, x, y)
    okg = O.ToeplitzOperator(og, ls, 1.0, sigma)
    ref = O.log_likelihood_gsgp(ost, okg, sigma, grid=og, x=x, solve_tol=1e-9, probes=30, max_depth=50,
                                quad_tol=0.0, seed=0, route="ski-operator", maxiter=5000)
    assert abs(r.const_term - ref["const_term"]) <= 1e-12 * abs(ref["const_term"])
    assert abs(r.quad_term - ref["quad_term"]) <= 1e-5 * abs(ref["quad_term"])
    assert abs(r.logdet_term - ref["logdet_term"]) <= 1e-5 * abs(ref["logdet_term"])
    assert abs(r.loglik - ref["loglik"]) <= 1e-5 * abs(ref["loglik"])
    # ill-conditioned data-fit solve (hundreds of iterations): count within 5 %
    assert abs(r.solver_iterations - ref["solver_iterations"]) <= max(1, 0.05 * ref["solver_iterations"])
    assert r.probes_used == 30
    # default quad_tol (0.01) early-stop path
    opts2 = G.LoglikOptions(solve_tol=1e-9, probes=30, slq=G.SlqOptions(max_depth=50, quad_tol=0.01), seed=0,
                            maxiter=5000)
    r2 = G.log_likelihood_gsgp(st, kg, sigma, opts2)
    ref2 = O.log_likelihood_gsgp(ost, okg, sigma, grid=og, x=x, solve_tol=1e-9, probes=30, max_depth=50,
                                 quad_tol=0.01, seed=0, route="ski-operator", maxiter=5000)
    assert abs(r2.loglik - ref2["loglik"]) <= 1e-5 * abs(ref2["loglik"])


def test_ski_route_requires_probe_images():
    g, x, y = make_case(n=2000)
    st = G.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
    spec = G.KernelSpec(G.Hyperparams(0.1, [0.2, 0.25, 0.3], 1.0))
    with pytest.raises(G.InvalidArgument, match="probe images"):
        G.log_likelihood_gsgp(st, G.ToeplitzOperator(g, spec), 0.1,
                              G.LoglikOptions(route=G.LogdetRoute.SkiOperator))


def _grid_case(d, sizes, ls, n=6000, sigma=0.1):
    g, x, y = make_case(d, sizes, n=n)
    st = G.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
    kg = G.ToeplitzOperator(g, G.KernelSpec(G.Hyperparams(sigma, ls, 1.0)))
    og = ogrid(g)
    ost = O.sufficient_stats(og, x, y)
    okg = O.ToeplitzOperator(og, ls, 1.0, sigma)
    return st, kg, ost, okg


@pytest.mark.parametrize("d,sizes,ls", [(1, (60,), [0.03]), (2, (16, 14), [0.2, 0.25]), (3, (8, 7, 6), [0.3, 0.3, 0.4])])
def test_symmetric_grid_route_matches_oracle(d, sizes, ls):
    """slq_logdet(K WᵀW K + σ²K) − slq_logdet(K) (gp.cpp:206-219) on identical m-dimensional
    probes: batched GPU Lanczos vs the oracle's sequential one.  Lengthscales keep K_G
    invertible in fp64 (cond ≤ 1e8); on a numerically singular K_G (e.g. ℓ = 0.1 on the 60-node
    1-D grid, cond ~1e301) SLQ(K) is rounding noise on either side — Auto routes those to
    Dense."""
    sigma = 0.1
    st, kg, ost, okg = _grid_case(d, sizes, ls, sigma=sigma)
    opts = G.LoglikOptions(solve_tol=1e-9, probes=6, slq=G.SlqOptions(max_depth=25, quad_tol=0.01), seed=3,
                           maxiter=5000, route=G.LogdetRoute.SymmetricGrid)
    r = G.log_likelihood_gsgp(st, kg, sigma, opts)
    ref = O.log_likelihood_gsgp(ost, okg, sigma, solve_tol=1e-9, probes=6, max_depth=25, quad_tol=0.01, seed=3,
                                route="symmetric-grid", maxiter=5000)
    assert r.logdet_route == ref["logdet_route"] == "symmetric-grid-slq"
    assert r.probes_used == ref["probes_used"] == 12
    assert abs(r.logdet_term - ref["logdet_term"]) <= 1e-6 * abs(ref["logdet_term"])
    assert abs(r.loglik - ref["loglik"]) <= 1e-6 * abs(ref["loglik"])


@pytest.mark.parametrize("d,sizes,ls", [(1, (80,), [0.1]), (2, (20, 18), [0.2, 0.25])])
def test_dense_route_matches_oracle(d, sizes, ls):
    """dense_logdet_grid_system (gp.cpp:116-140): LU with partial pivoting of K WᵀW + σ²I."""
    sigma = 0.1
    st, kg, ost, okg = _grid_case(d, sizes, ls, sigma=sigma)
    opts = G.LoglikOptions(solve_tol=1e-9, maxiter=5000, route=G.LogdetRoute.Dense)
    r = G.log_likelihood_gsgp(st, kg, sigma, opts)
    ref = O.log_likelihood_gsgp(ost, okg, sigma, solve_tol=1e-9, route="dense", maxiter=5000)
    assert r.logdet_route == "dense"
    assert abs(r.logdet_term - ref["logdet_term"]) <= 1e-9 * abs(ref["logdet_term"])
    # the quadratic term (yᵀy − wᵀz̄)/σ² cancels: its agreement is set by the 1e-9 data-fit solve
    assert abs(r.quad_term - ref["quad_term"]) <= 1e-5 * abs(ref["quad_term"])
    assert abs(r.loglik - ref["loglik"]) <= 1e-6 * abs(ref["loglik"])
    with pytest.raises(G.InvalidArgument, match="too large for the dense"):
        G.log_likelihood_gsgp(st, kg, sigma, G.LoglikOptions(solve_tol=1e-9, maxiter=5000, route=G.LogdetRoute.Dense,
                                                             dense_cap=10))


def test_auto_route_selection_matches_oracle():
    """Auto (gp.cpp:181-205): Dense when cond(K_G) > 1e8 and m ≤ dense_cap, else SymmetricGrid;
    SkiOperator whenever the statistics carry probe images."""
    sigma = 0.1
    # long lengthscale on a fine 1-D grid: K_G is numerically singular → dense
    st, kg, ost, okg = _grid_case(1, (120,), [0.5], sigma=sigma)
    r = G.log_likelihood_gsgp(st, kg, sigma, G.LoglikOptions(solve_tol=1e-9, maxiter=20000))
    ref = O.log_likelihood_gsgp(ost, okg, sigma, solve_tol=1e-9, maxiter=20000)
    assert r.logdet_route == ref["logdet_route"] == "dense"
    assert abs(r.loglik - ref["loglik"]) <= 1e-6 * abs(ref["loglik"])
    # short lengthscale: well conditioned → symmetric grid
    st, kg, ost, okg = _grid_case(2, (12, 11), [0.1, 0.1], sigma=sigma)
    r = G.log_likelihood_gsgp(st, kg, sigma, G.LoglikOptions(solve_tol=1e-9, probes=4, maxiter=5000))
    ref = O.log_likelihood_gsgp(ost, okg, sigma, solve_tol=1e-9, probes=4, maxiter=5000)
    assert r.logdet_route == ref["logdet_route"] == "symmetric-grid-slq"
