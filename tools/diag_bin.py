"""Diagnostics: time the binning phases of the config-3 precompute (phase timers)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_11751_b200 as G  # noqa: E402
from paper_2101_11751_b200 import synthetic as S  # noqa: E402

cfg = S.CONFIGS[3]
ctx = G.Context(0)
rows = S.generate_torch(3, device="cuda")
if len(sys.argv) > 1 and sys.argv[1] == "shuffled_uniform":
    rows[:, :3] = torch.rand((rows.shape[0], 3), device="cuda", dtype=torch.float32) * 0.9 + 0.05
grid = S.grid_for(cfg)
acc = G.SufficientStatsAccumulator(grid, ctx=ctx)
for _ in range(2):
    acc.reset(); acc.add(rows); acc.finalize()
ctx.enable_phase_timing(True)
ctx.reset_phase_times()
for _ in range(3):
    acc.reset(); acc.add(rows); acc.finalize()
print(os.environ.get("GSGPC_DIAG_BIN", "0"), sys.argv[1:], {k: round(v[0] / v[1], 3) for k, v in ctx.phase_times().items()})
