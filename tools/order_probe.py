"""Diagnostic: run a test file in-process, then config 5 statistics; report Σ W^T y vs Σ y."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import pytest  # noqa: E402

sel = (sys.argv[1] if len(sys.argv) > 1 else "tests/test_gpu_ingest.py").split(",")
kexpr = sys.argv[2] if len(sys.argv) > 2 else ""
args = ["-q", "-p", "no:cacheprovider"] + sel + (["-k", kexpr] if kexpr else [])
pytest.main(args)
import numpy as np  # noqa: E402
import paper_2101_11751_b200 as G  # noqa: E402
from paper_2101_11751_b200 import synthetic as S  # noqa: E402

cfg = S.CONFIGS[5]
rows = S.generate_torch(5, device="cuda")
g = S.grid_for(cfg)
ws = []
for rep in range(2):
    gs = G.sufficient_stats(g, G.InterpScheme.Cubic, rows)
    ysum = rows[:, 3].sum().item()
    w = gs.wty()
    ws.append(w)
    vals, _ = gs.stencil()
    yty = (rows[:, 3] ** 2).sum().item()
    print(f"rep {rep}: sum wty {w.sum():.6e} sum y {ysum:.6e} | WtW total {vals[0].sum() + 2 * vals[1:].sum():.6e} "
          f"n {gs.n()} yty {gs.yty():.6e} vs {yty:.6e}", flush=True)
d = np.abs(ws[0] - ws[1]).reshape(g.size(0), -1).max(axis=1)
bad = np.nonzero(d > 1e-9 * np.abs(ws[1]).max())[0]
print("planes differing:", len(bad), bad[:20], bad[-5:] if len(bad) else "")
flat = np.nonzero(np.abs(ws[0] - ws[1]) > 1e-9 * np.abs(ws[1]).max())[0]
print("nodes differing:", len(flat), flat[:5], flat[-5:] if len(flat) else "", "of", ws[0].size)
print("ratio rep0/rep1 on differing:", (ws[0][flat] / np.where(ws[1][flat] == 0, 1, ws[1][flat]))[:8] if len(flat) else "")
