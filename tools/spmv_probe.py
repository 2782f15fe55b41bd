"""Standalone W^T W stencil SpMV (k_spmv via SufficientStats.apply_wtw) on the full statistics
of a config, timed with CUDA events; for ncu captures of the SpMV alone."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2101_11751_b200 as G  # noqa: E402
from paper_2101_11751_b200 import synthetic as S  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = S.CONFIGS[cfg_id]
ctx = G.Context(0)
rows = S.generate_torch(cfg_id, device="cuda")
st = G.sufficient_stats(S.grid_for(cfg), G.InterpScheme.Cubic, rows, ctx=ctx)
del rows
torch.cuda.empty_cache()
m = S.grid_for(cfg).num_points()
v = torch.randn(m, dtype=torch.float64, device="cuda")
out = torch.empty_like(v)
ext = torch.cuda.ExternalStream(ctx.stream)
for _ in range(3):
    st.apply_wtw(v, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(ext)
for _ in range(reps):
    st.apply_wtw(v, out=out)
e1.record(ext)
e1.synchronize()
print(f"config {cfg_id}: SpMV {e0.elapsed_time(e1) / reps * 1e3:.1f} us per call (incl. API overhead)")
