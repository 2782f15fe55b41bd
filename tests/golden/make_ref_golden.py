"""Generate tests/golden/ref_golden.json FROM THE REFERENCE'S OWN CODE (committed; rerun here to
refresh: needs /root/reference, which `oracle.ref` compiles against the stand-in headers of
oracle/refshim — see its README.md).

The fixture travels where neither /root/reference nor oracle/_ref exist.  It holds, for inputs
that the tests regenerate from fixed seeds:

* weights     — interp_weights (interp.cpp:79-134) of hand-picked points: indices and values.
* configs     — the BASELINE configurations' grids and synthetic value distributions
                (paper_2101_11751_b200.synthetic, numpy streams) on deterministic prefixes:
                n, nnz, max_row_nnz, yᵀy, a SHA-256 of the CSR structure (row_ptr ‖ col as
                int64), and linear functionals of W^T W and W^T y.
* solve       — a well-conditioned 2-D system solved tightly (so that the answer, not the stopping
                iterate, is compared): leading α/β/ρ of factorized_cg_grid_rhs
                (solvers.cpp:271-336), the posterior mean coefficients (gp.cpp:326-352),
                predictions, and log_likelihood_gsgp (gp.cpp:158-240) per log-det route.
* probes      — rademacher_probe (gp.cpp:16-25): leading signs per (seed, probe).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

CONFIG_PREFIX = {1: 20000, 2: 20000, 3: 3000, 5: 3000}


def probe_vectors(m):
    i = np.arange(m, dtype=np.float64)
    return np.cos(0.37 * i + 0.1), np.sin(0.11 * i + 0.2)


def struct_hash(rp, col):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(rp, np.int64).tobytes())
    h.update(np.ascontiguousarray(col, np.int64).tobytes())
    return h.hexdigest()


def weight_points():
    """(d, sizes, scheme, x) cases: interior, on-node, snap band, data bounds."""
    out = []
    for d, sizes in ((1, [12]), (2, [9, 11]), (3, [8, 7, 9])):
        rng = np.random.default_rng(40 + d)
        for scheme in (0, 1):
            pts = [rng.random(d) for _ in range(4)]
            pts += [np.zeros(d), np.ones(d), np.full(d, 0.5), np.full(d, 0.25 + 3e-10), np.full(d, 0.75 - 5e-10)]
            for x in pts:
                out.append((d, sizes, scheme, [float(v) for v in x]))
    return out


def solve_inputs():
    rng = np.random.default_rng(77)
    n, d, sizes = 6000, 2, [20, 17]
    x = rng.random((n, d))
    y = np.sin(4.0 * x.sum(axis=1)) + 0.1 * rng.standard_normal(n)
    ls = [1.3 / (s - 5) for s in sizes]
    return x, y, sizes, ls, 1.2, 0.1


def main():
    import oracle.ref as R
    from paper_2101_11751_b200 import synthetic as S

    assert R.available(), "oracle/_ref/libgsgp_ref.so cannot be built (needs /root/reference)"
    gold = {"made_by": "tests/golden/make_ref_golden.py", "source": R.ref_build_info(), "weights": [], "configs": {},
            "probes": []}
    for d, sizes, scheme, x in weight_points():
        g = R.fit_grid_to_data([0.0] * d, [1.0] * d, sizes, scheme)
        idx, w = R.interp_weights(g, x, scheme)
        gold["weights"].append({"d": d, "sizes": sizes, "scheme": scheme, "x": x, "idx": [int(i) for i in idx],
                                "w": [float(v) for v in w]})
    for cid, n in CONFIG_PREFIX.items():
        cfg = S.CONFIGS[cid]
        x, y = S.generate(cid, n=n)
        g = S.grid_for(cfg)
        og = R.Grid([g.min(k) for k in range(cfg.d)], [g.max(k) for k in range(cfg.d)],
                    [g.size(k) for k in range(cfg.d)])
        st = R.sufficient_stats(og, np.asarray(x, np.float64), np.asarray(y, np.float64), scheme=1)
        rp, col, val, wty = st.csr()
        v1, v2 = probe_vectors(st.m)
        gold["configs"][str(cid)] = {
            "n": int(st.n), "m": int(st.m), "nnz": int(st.nnz), "max_row_nnz": st.max_row_nnz(), "yty": st.yty,
            "structure_sha256": struct_hash(rp, col), "val_sum": float(val.sum()), "val_abs_max": float(np.abs(val).max()),
            "v2_A_v1": float(v2 @ st.apply_wtw(v1)), "v1_A_v1": float(v1 @ st.apply_wtw(v1)),
            "wty_v1": float(wty @ v1), "wty_v2": float(wty @ v2), "wty_sq": float(wty @ wty)}
    x, y, sizes, ls, oscale, sigma = solve_inputs()
    g = R.fit_grid_to_data([0.0, 0.0], [1.0, 1.0], sizes, 1)
    st = R.sufficient_stats(g, x, y)
    kg = R.ToeplitzOperator(g, ls, oscale, sigma)
    r0 = -kg.apply(st.wty) / sigma ** 2
    cg = R.factorized_cg_grid_rhs(kg, st, r0, sigma, rel_tol=1e-10, maxiter=4000)
    mean, iters, _ = R.posterior_mean_gsgp(kg, st, sigma, 1e-9, 6000)
    pts = np.random.default_rng(78).random((50, 2))
    sol = {"sizes": sizes, "lengthscales": ls, "outputscale": oscale, "sigma": sigma, "kg_r0_sq": float(r0 @ r0),
           "cg_iterations": cg.iterations, "alphas": [float(v) for v in cg.alphas[:10]],
           "betas": [float(v) for v in cg.betas[:10]], "rho": [float(v) for v in cg.residual_trace[:10]],
           "xhat_d": [float(v) for v in cg.xhat_d], "mean_iterations": iters, "mean_coeffs": [float(v) for v in mean],
           "pred": [float(v) for v in R.predict_mean(g, mean, pts)], "loglik": {}}
    for route, with_w in (("ski-operator", True), ("symmetric-grid", False), ("dense", False)):
        ll = R.log_likelihood_gsgp(st, kg, sigma, grid=g, x=x if with_w else None, solve_tol=1e-9, probes=8,
                                   max_depth=40, quad_tol=0.0, seed=5, route=route, maxiter=4000)
        sol["loglik"][route] = {k: (float(v) if isinstance(v, float) else v) for k, v in ll.items()}
    gold["solve"] = sol
    for seed, p in ((0, 0), (5, 3), (2 ** 40 + 5, 29), (123456789, 2 ** 33)):
        v = R.rademacher_probe(256, seed, p)
        gold["probes"].append({"seed": seed, "probe": p, "plus": "".join("1" if s > 0 else "0" for s in v)})
    with open(os.path.join(HERE, "ref_golden.json"), "w") as f:
        json.dump(gold, f)
    print("wrote ref_golden.json", os.path.getsize(os.path.join(HERE, "ref_golden.json")), "bytes")


if __name__ == "__main__":
    main()
