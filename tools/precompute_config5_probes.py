"""Config 5 precompute with 30 seeded probe streams: per-phase device times (probe RNG included
in the moments/scatter phases) and the wall time of one reset + add + finalize."""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_2101_11751_b200 as G  # noqa: E402
from paper_2101_11751_b200 import synthetic as S  # noqa: E402

cfg = S.CONFIGS[5]
ctx = G.Context(0)
rows = S.generate_torch(5, device="cuda")
grid = S.grid_for(cfg)
acc = G.SufficientStatsAccumulator(grid, G.InterpScheme.Cubic, ctx=ctx)
acc.enable_probes(30, seed=0)
out = {}
for rep in range(4):
    acc.reset()
    ctx.synchronize()
    t0 = time.perf_counter()
    acc.add(rows)
    st = acc.finalize()
    ctx.synchronize()
    out[f"step{rep}_ms"] = 1e3 * (time.perf_counter() - t0)
ctx.enable_phase_timing(True)
ctx.reset_phase_times()
acc.reset()
acc.add(rows)
st = acc.finalize()
ctx.synchronize()
out["phases_ms"] = {k: v[0] for k, v in ctx.phase_times().items()}
print(json.dumps(out))
