"""Where do the GPU and oracle CG traces part on config 3 (1e6-row prefix, identical statistics)?
Per-iteration relative α differences (GPU vs oracle FFT, oracle direct-K_G vs FFT), the SpMV
difference on identical statistics, and stored-but-untouched stencil entries."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
import paper_2101_11751_b200 as G  # noqa: E402
from paper_2101_11751_b200 import synthetic as S  # noqa: E402
from helpers import csr_to_half_stencil, oracle_stats_from_gpu  # noqa: E402

O.set_threads(os.cpu_count() or 8)
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
cfg = S.CONFIGS[cid]
g = S.grid_for(cfg)
og = O.Grid([g.min(k) for k in range(g.dim())], [g.max(k) for k in range(g.dim())], list(cfg.sizes))
x, y = S.generate(cid, n)
gst = G.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
ost = oracle_stats_from_gpu(gst)
out = {}
vals, _ = gst.stencil()
rp, col, val, wty = ost.csr()
exp = csr_to_half_stencil(rp, col, val, list(cfg.sizes), 4)
mask = exp != 0
out["stencil_internal_vs_export_max"] = float(np.abs(vals - exp).max())
out["untouched_nonzero_count"] = int(((vals != 0) & ~mask).sum())
out["untouched_nonzero_max"] = float(np.abs(vals[~mask]).max()) if (~mask).any() else 0.0
rng = np.random.default_rng(0)
v = rng.standard_normal(g.num_points())
a, b = gst.apply_wtw(v), ost.apply_wtw(v)
out["spmv_rel_entry"] = float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))
out["spmv_rel_norm"] = float(np.abs(a - b).max() / np.abs(b).max())
spec = S.kernel_for(cfg)
kg = G.ToeplitzOperator(g, spec)
okg = O.ToeplitzOperator(og, list(cfg.lengthscales), cfg.outputscale, cfg.noise_std)
okd = O.ToeplitzOperator(og, list(cfg.lengthscales), cfg.outputscale, cfg.noise_std)
okd.set_direct()
kv, ov = kg.apply(v), okg.apply(v)
out["kg_rel_entry_p99"] = float(np.quantile(np.abs(kv - ov) / np.maximum(np.abs(ov), 1e-300), 0.99))
r0 = -okg.apply(wty) / cfg.noise_variance
it = 40
ores = O.factorized_cg_grid_rhs(okg, ost, r0, cfg.noise_std, eps_abs=1e-30, maxiter=it)
dres = O.factorized_cg_grid_rhs(okd, ost, r0, cfg.noise_std, eps_abs=1e-30, maxiter=it)
gres = G.factorized_cg_grid_rhs(kg, gst, r0, cfg.noise_std, G.GridRhsTolerance(eps_abs=1e-30), it)
ra = ores.alphas
out["alpha_rel_gpu"] = [float(abs(p - q) / abs(q)) for p, q in zip(gres.alphas, ra)]
out["alpha_rel_direct"] = [float(abs(p - q) / abs(q)) for p, q in zip(dres.alphas, ra)]
out["rho_rel_gpu"] = [float(abs(p - q) / abs(q)) for p, q in zip(gres.residual_trace, ores.residual_trace)]
print(json.dumps(out))
