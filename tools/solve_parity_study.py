"""Solve parity on the BASELINE configurations on IDENTICAL statistics (GPU box tool).

Config 1 (full n): the oracle's own statistics → GSGPSST1 → gsgpc_stats_load, then the
posterior mean on both sides; configs 2, 3 (prefix), 5 (prefix): the GPU's statistics →
CSR → oracle, then fixed-window CG traces / the log-likelihood.  The oracle also runs with
its K_G applied by direct Toeplitz sums (same operator, another rounding) to measure how far
the solve moves under O(1e-16) perturbations alone.  Prints one JSON object.
"""
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
import paper_2101_11751_b200 as G  # noqa: E402
from paper_2101_11751_b200 import synthetic as S  # noqa: E402
from helpers import oracle_stats_from_gpu, write_gsgpsst1  # noqa: E402

O.set_threads(os.cpu_count() or 8)
out = {"threads": os.cpu_count()}
which = sys.argv[1:] or ["1", "2", "3", "5"]


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def ogrid(g):
    return O.Grid([g.min(k) for k in range(g.dim())], [g.max(k) for k in range(g.dim())],
                  [g.size(k) for k in range(g.dim())])


if "1" in which:
    cfg = S.CONFIGS[1]
    g = S.grid_for(cfg)
    og = ogrid(g)
    x, y = S.generate(1)
    t = time.time()
    ost = O.sufficient_stats(og, x, y, nthreads=os.cpu_count() or 8)
    rp, col, val, wty = ost.csr()
    p = os.path.join(tempfile.mkdtemp(), "c1.gsgpsst")
    write_gsgpsst1(p, (og.mins, og.maxs, og.sizes), 1, rp, col, val, wty, ost.yty, ost.n)
    gst = G.load_stats(p).stats
    spec = S.kernel_for(cfg)
    kg = G.ToeplitzOperator(g, spec)
    okg = O.ToeplitzOperator(og, list(cfg.lengthscales), cfg.outputscale, cfg.noise_std)
    okd = O.ToeplitzOperator(og, list(cfg.lengthscales), cfg.outputscale, cfg.noise_std)
    okd.set_direct()
    r = {}
    for tol in (1e-6, 1e-8):
        omc, oit, _ = O.posterior_mean_gsgp(okg, ost, cfg.noise_std, tol, 5000)
        dmc, dit, _ = O.posterior_mean_gsgp(okd, ost, cfg.noise_std, tol, 5000)
        model = G.posterior_mean_gsgp(gst, kg, spec, G.InterpScheme.Cubic, cfg.noise_std, tol, 5000)
        tp = np.linspace(-10.0, 10.0, 1000).reshape(-1, 1)
        op = O.predict_mean(og, omc, tp)
        r[str(tol)] = {
            "iters_oracle_fft": oit, "iters_oracle_direct": dit, "iters_gpu": model.solve_iterations,
            "mean_gpu_vs_fft": rel(model.mean_coeffs, omc), "mean_direct_vs_fft": rel(dmc, omc),
            "pred_gpu_vs_fft": rel(model.predict_mean(tp), op),
            "pred_direct_vs_fft": rel(O.predict_mean(og, dmc, tp), op),
        }
    # fixed-window traces on identical statistics
    r0 = -okg.apply(wty) / cfg.noise_variance
    eps = 1e-30
    ores = O.factorized_cg_grid_rhs(okg, ost, r0, cfg.noise_std, eps_abs=eps, maxiter=100)
    dres = O.factorized_cg_grid_rhs(okd, ost, r0, cfg.noise_std, eps_abs=eps, maxiter=100)
    gres = G.factorized_cg_grid_rhs(kg, gst, r0, cfg.noise_std, G.GridRhsTolerance(eps_abs=eps), 100)
    for name, res in (("gpu", gres), ("direct", dres)):
        for w in (20, 50, 100):
            r[f"alpha{w}_{name}"] = rel(res.alphas[:w], ores.alphas[:w])
            r[f"rho{w}_{name}"] = rel(res.residual_trace[:w], ores.residual_trace[:w])
        r[f"xhat100_{name}"] = rel(res.xhat_d, ores.xhat_d)
    r["seconds"] = time.time() - t
    out["config1"] = r
    print(json.dumps(out), flush=True)

for cid, n in (("2", None), ("3", 1_000_000)):
    if cid not in which:
        continue
    t = time.time()
    cfg = S.CONFIGS[int(cid)]
    g = S.grid_for(cfg)
    og = ogrid(g)
    rows = S.generate_torch(int(cid), n, device="cuda")
    gst = G.sufficient_stats(g, G.InterpScheme.Cubic, rows)
    del rows
    ost = oracle_stats_from_gpu(gst)
    spec = S.kernel_for(cfg)
    kg = G.ToeplitzOperator(g, spec)
    okg = O.ToeplitzOperator(og, list(cfg.lengthscales), cfg.outputscale, cfg.noise_std)
    okd = O.ToeplitzOperator(og, list(cfg.lengthscales), cfg.outputscale, cfg.noise_std)
    okd.set_direct()
    wty = gst.wty()
    r0 = -okg.apply(wty) / cfg.noise_variance
    r = {"kg_apply_gpu_vs_fft": rel(kg.apply(wty), okg.apply(wty))}
    eps = 1e-30
    ores = O.factorized_cg_grid_rhs(okg, ost, r0, cfg.noise_std, eps_abs=eps, maxiter=100)
    dres = O.factorized_cg_grid_rhs(okd, ost, r0, cfg.noise_std, eps_abs=eps, maxiter=100)
    gres = G.factorized_cg_grid_rhs(kg, gst, r0, cfg.noise_std, G.GridRhsTolerance(eps_abs=eps), 100)
    for name, res in (("gpu", gres), ("direct", dres)):
        for w in (20, 50, 100):
            r[f"alpha{w}_{name}"] = rel(res.alphas[:w], ores.alphas[:w])
            r[f"beta{w}_{name}"] = rel(res.betas[:w], ores.betas[:w])
            r[f"rho{w}_{name}"] = rel(res.residual_trace[:w], ores.residual_trace[:w])
        r[f"xhat100_{name}"] = rel(res.xhat_d, ores.xhat_d)
    r["oracle_seconds_100it"] = ores.loop_seconds
    r["seconds"] = time.time() - t
    out["config" + cid] = r
    print(json.dumps(out), flush=True)

if "5" in which:
    t = time.time()
    cfg = S.CONFIGS[5]
    g = S.grid_for(cfg)
    og = ogrid(g)
    n = int(os.environ.get("C5N", "1000000"))
    P = int(os.environ.get("C5P", "30"))
    rows = S.generate_torch(5, n, device="cuda")
    acc = G.SufficientStatsAccumulator(g)
    acc.enable_probes(P, 0)
    acc.add(rows)
    gst = acc.finalize()
    host = rows.cpu().numpy()
    del rows
    ost = oracle_stats_from_gpu(gst)
    spec = S.kernel_for(cfg)
    kg = G.ToeplitzOperator(g, spec)
    okg = O.ToeplitzOperator(og, list(cfg.lengthscales), cfg.outputscale, cfg.noise_std)
    r = {"n": n, "probes": P}
    for stol in (1e-8,):
        opts = G.LoglikOptions(solve_tol=stol, probes=P, slq=G.SlqOptions(50, 0.0), seed=0, maxiter=20000,
                               route=G.LogdetRoute.SkiOperator)
        t1 = time.time()
        gl = G.log_likelihood_gsgp(gst, kg, cfg.noise_std, opts)
        tg = time.time() - t1
        t1 = time.time()
        ol = O.log_likelihood_gsgp(ost, okg, cfg.noise_std, grid=og, x=host[:, :3], solve_tol=stol, probes=P,
                                   max_depth=50, quad_tol=0.0, seed=0, route="ski-operator", maxiter=20000)
        to = time.time() - t1
        r[str(stol)] = {"gpu": [gl.loglik, gl.logdet_term, gl.quad_term, gl.const_term, gl.solver_iterations],
                        "oracle": ol, "gpu_s": tg, "oracle_s": to}
    r["seconds"] = time.time() - t
    out["config5"] = r
    print(json.dumps(out, default=str), flush=True)
