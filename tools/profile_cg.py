"""Profiling driver: config-3 precompute once, then N EFCG iterations (for ncu -k filters)."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_11751_b200 as G  # noqa: E402
from paper_2101_11751_b200 import synthetic as S  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cfg = S.CONFIGS[cfg_id]
ctx = G.Context(0)
rows = S.generate_torch(cfg_id, device="cuda")
grid = S.grid_for(cfg)
spec = S.kernel_for(cfg)
st = G.sufficient_stats(grid, G.InterpScheme.Cubic, rows, ctx=ctx)
del rows
torch.cuda.empty_cache()
kg = G.ToeplitzOperator(grid, spec, ctx=ctx)
s2 = cfg.noise_std ** 2
r0 = -kg.apply(st.wty()) / s2
res = G.factorized_cg_grid_rhs(kg, st, r0, cfg.noise_std, G.GridRhsTolerance(eps_abs=0.0), iters)
print("iters", res.iterations, "ms/iter", 1e3 * res.loop_seconds / max(res.iterations, 1))
print("dmma/mixed TFLOP/s", ctx.fp64_tensor_tflops(), "dfma", ctx.fp64_peak_tflops())
