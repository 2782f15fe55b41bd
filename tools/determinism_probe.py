"""Run-to-run reproducibility probe (config 5 size): two precomputes of the same rows, then
the data-fit EFCG of log_likelihood_gsgp (eps_abs = tol²·yᵀy) on each, and twice on the same
statistics.  Prints the stencil difference and the solver outcomes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2101_11751_b200 as G  # noqa: E402
from paper_2101_11751_b200 import synthetic as S  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = S.CONFIGS[cfg_id]
ctx = G.Context(0)
rows = S.generate_torch(cfg_id, device="cuda")
grid = S.grid_for(cfg)
spec = S.kernel_for(cfg)
stats = [G.sufficient_stats(grid, G.InterpScheme.Cubic, rows, ctx=ctx) for _ in range(2)]
a, _ = stats[0].stencil()
b, _ = stats[1].stencil()
print("stencil max |diff| / max |a|:", float(np.abs(a - b).max() / np.abs(a).max()),
      "identical:", bool(np.array_equal(a, b)))
kg = G.ToeplitzOperator(grid, spec, ctx=ctx)
s2 = cfg.noise_std ** 2
for i, st in enumerate(stats + [stats[0]]):
    wty = st.wty()
    r0 = -kg.apply(wty) / s2
    tol = G.GridRhsTolerance(eps_abs=cfg.tol * cfg.tol * st.yty())
    res = G.factorized_cg_grid_rhs(kg, st, r0, cfg.noise_std, tol, 20000)
    zbar = kg.apply(np.asarray(res.xhat_d) + wty / s2)
    quad = (st.yty() - float(wty @ zbar)) / s2
    print(f"stats {i if i < 2 else 0}: iterations {res.iterations} converged {res.converged} quad {quad:.9e} "
          f"rho {res.residual_sq:.3e}", flush=True)
