"""Config 5 (log-likelihood workload) at full size: precompute with 30 probe images, then
log_likelihood_gsgp on the SkiOperator route.  Timing probe."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_11751_b200 as G  # noqa: E402
from paper_2101_11751_b200 import synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else None
cfg = S.CONFIGS[5]
ctx = G.Context(0)
rows = S.generate_torch(5, n, device="cuda")
grid = S.grid_for(cfg)
spec = S.kernel_for(cfg)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    acc = G.SufficientStatsAccumulator(grid, G.InterpScheme.Cubic, ctx=ctx)
    acc.enable_probes(30, seed=0)
    acc.add(rows)
    st = acc.finalize()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    kg = G.ToeplitzOperator(grid, spec, ctx=ctx)
    opts = G.LoglikOptions(solve_tol=cfg.tol, probes=30, slq=G.SlqOptions(max_depth=50, quad_tol=0.0), seed=0,
                           maxiter=20000)
    r = G.log_likelihood_gsgp(st, kg, cfg.noise_std, opts)
    t2 = time.perf_counter()
    print(f"n={rows.shape[0]} precompute+probes {1e3 * (t1 - t0):.1f} ms ({rows.shape[0] / (t1 - t0) / 1e9:.2f}e9 rows/s)"
          f"  loglik {1e3 * (t2 - t1):.1f} ms  route {r.logdet_route} loglik {r.loglik:.6e} logdet {r.logdet_term:.6e} "
          f"quad {r.quad_term:.6e} cg_iters {r.solver_iterations}", flush=True)
