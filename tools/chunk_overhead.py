"""Diagnostics: cost of splitting one device-resident precompute into k add() calls
(each call bins and flushes every cell's moments once)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_11751_b200 as G  # noqa: E402
from paper_2101_11751_b200 import synthetic as S  # noqa: E402

cfg = S.CONFIGS[3]
ctx = G.Context(0)
rows = S.generate_torch(3, device="cuda")
grid = S.grid_for(cfg)
acc = G.SufficientStatsAccumulator(grid, G.InterpScheme.Cubic, ctx=ctx)
n = rows.shape[0]
for parts in (1, 2, 4, 8, 16):
    best = 1e9
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        acc.reset()
        step = (n + parts - 1) // parts
        for a0 in range(0, n, step):
            acc.add(rows[a0:a0 + step])
        ctx.synchronize()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{parts:2d} add() calls: {best:.2f} ms  ({(best) / parts:.2f} ms per call)", flush=True)
