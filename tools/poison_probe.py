"""Diagnostic: config statistics with the finalize workspace NaN-poisoned (GSGPC_DEBUG_POISON_WS=1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2101_11751_b200 as G  # noqa: E402
from paper_2101_11751_b200 import synthetic as S  # noqa: E402

for cfg_id, n in [(5, 2_000_000), (3, 2_000_000), (2, 2_000_000), (4, 2_000_000)]:
    cfg = S.CONFIGS[cfg_id]
    rows = S.generate_torch(cfg_id, n, device="cuda")
    g = S.grid_for(cfg)
    gs = G.sufficient_stats(g, G.InterpScheme.Cubic, rows)
    w = gs.wty()
    v, _ = gs.stencil()
    print(cfg_id, "wty nan", int(np.isnan(w).sum()), "sum", w.sum(), "vs", rows[:, cfg.d].sum().item(),
          "| stencil nan", int(np.isnan(v).sum()), flush=True)
