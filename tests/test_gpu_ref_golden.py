"""The CUDA path against tests/golden/ref_golden.json — outputs of the REFERENCE'S OWN CODE
(tests/golden/make_ref_golden.py, through oracle.ref), on inputs regenerated from fixed seeds.
Bounds: indices, counts and the CSR structure exact; weights bit-exact; statistics 1e-10;
leading CG scalars 1e-8; mean coefficients, predictions and log-likelihood terms 1e-5."""
import json
import os
import sys

import numpy as np
import pytest

import paper_2101_11751_b200 as G

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_ref_golden as MG  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(HERE, "golden", "ref_golden.json")))


def test_weights_bit_exact():
    for w in GOLD["weights"]:
        scheme = G.InterpScheme(w["scheme"])
        g = G.fit_grid_to_data(np.zeros(w["d"]), np.ones(w["d"]), w["sizes"], scheme)
        idx, val = G.interp_weights(g, np.array(w["x"]), scheme)
        assert [int(i) for i in idx] == w["idx"]
        assert [float(v) for v in val] == w["w"]


@pytest.mark.parametrize("cid", sorted(MG.CONFIG_PREFIX))
def test_baseline_config_statistics(cid):
    from paper_2101_11751_b200 import synthetic as S

    gold = GOLD["configs"][str(cid)]
    cfg = S.CONFIGS[cid]
    x, y = S.generate(cid, n=MG.CONFIG_PREFIX[cid])
    st = G.sufficient_stats(S.grid_for(cfg), G.InterpScheme.Cubic, x, y)
    rp, col, val = st.csr()
    m = st.grid_size()
    v1, v2 = MG.probe_vectors(m)
    assert (st.n(), m, len(val), st.max_row_nnz()) == (gold["n"], gold["m"], gold["nnz"], gold["max_row_nnz"])
    assert MG.struct_hash(rp, col) == gold["structure_sha256"]
    assert abs(st.yty() - gold["yty"]) <= 1e-12 * gold["yty"]
    scale = gold["val_abs_max"]
    assert abs(float(np.abs(val).max()) - scale) <= 1e-10 * scale
    # linear functionals of W^T W and W^T y, against sums of |terms| of the same size
    a11 = float(v1 @ st.apply_wtw(v1))
    assert abs(a11 - gold["v1_A_v1"]) <= 1e-10 * abs(gold["v1_A_v1"])
    assert abs(float(v2 @ st.apply_wtw(v1)) - gold["v2_A_v1"]) <= 1e-10 * abs(gold["v1_A_v1"])
    wty = st.wty()
    assert abs(float(wty @ wty) - gold["wty_sq"]) <= 1e-10 * gold["wty_sq"]
    assert abs(float(wty @ v1) - gold["wty_v1"]) <= 1e-10 * np.sqrt(gold["wty_sq"] * m)


def test_solve_and_loglik():
    sol = GOLD["solve"]
    x, y, sizes, ls, oscale, sigma = MG.solve_inputs()
    g = G.fit_grid_to_data(np.zeros(2), np.ones(2), sizes, G.InterpScheme.Cubic)
    spec = G.KernelSpec(G.Hyperparams(sigma, ls, oscale))
    acc = G.SufficientStatsAccumulator(g)
    acc.enable_probes(8, seed=5)
    acc.add(x, y)
    st = acc.finalize()
    kg = G.ToeplitzOperator(g, spec)
    r0 = -kg.apply(st.wty()) / sigma ** 2
    assert float(r0 @ r0) == pytest.approx(sol["kg_r0_sq"], rel=1e-10)
    cg = G.factorized_cg_grid_rhs(kg, st, r0, sigma, G.GridRhsTolerance(rel_tol=1e-10), 4000)
    assert np.allclose(cg.alphas[:10], sol["alphas"], rtol=1e-8, atol=0)
    assert np.allclose(cg.betas[:10], sol["betas"], rtol=1e-8, atol=0)
    assert np.allclose(cg.residual_trace[:10], sol["rho"], rtol=1e-8, atol=0)
    assert abs(cg.iterations - sol["cg_iterations"]) <= max(3, sol["cg_iterations"] // 40)  # round-off drift
    xd = np.array(sol["xhat_d"])
    assert np.abs(cg.xhat_d - xd).max() <= 1e-5 * np.abs(xd).max()
    model = G.posterior_mean_gsgp(st, kg, spec, G.InterpScheme.Cubic, sigma, 1e-9, 6000)
    mc = np.array(sol["mean_coeffs"])
    assert np.abs(model.mean_coeffs - mc).max() <= 1e-5 * np.abs(mc).max()
    assert abs(model.solve_iterations - sol["mean_iterations"]) <= max(3, sol["mean_iterations"] // 40)
    pts = np.random.default_rng(78).random((50, 2))
    pred = np.array(sol["pred"])
    assert np.abs(model.predict_mean(pts) - pred).max() <= 1e-5 * np.abs(pred).max()
    for route, key in ((G.LogdetRoute.SkiOperator, "ski-operator"), (G.LogdetRoute.SymmetricGrid, "symmetric-grid"),
                       (G.LogdetRoute.Dense, "dense")):
        opts = G.LoglikOptions(solve_tol=1e-9, probes=8, slq=G.SlqOptions(max_depth=40, quad_tol=0.0), seed=5,
                               maxiter=4000, route=route)
        r = G.log_likelihood_gsgp(st, kg, sigma, opts)
        ref = sol["loglik"][key]
        tol = 1e-4 if key == "symmetric-grid" else 1e-5
        assert r.logdet_route == ref["logdet_route"]
        assert abs(r.const_term - ref["const_term"]) <= 1e-12 * abs(ref["const_term"])
        assert abs(r.quad_term - ref["quad_term"]) <= 1e-5 * abs(ref["quad_term"])
        assert abs(r.loglik - ref["loglik"]) <= tol * abs(ref["loglik"])


def test_probe_signs_bit_exact():
    for p in GOLD["probes"]:
        if p["probe"] >= 2 ** 31:
            continue  # the library takes probe indices as int
        bits = G.probe_stream_bits(p["seed"], p["probe"], 0, 256)
        assert "".join("1" if b else "0" for b in bits) == p["plus"]
