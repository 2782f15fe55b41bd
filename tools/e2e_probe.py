"""Where the end-to-end (pinned host rows) precompute step spends its time (diagnostics)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_11751_b200 as G  # noqa: E402
from paper_2101_11751_b200 import synthetic as S  # noqa: E402

cfg = S.CONFIGS[3]
ctx = G.Context(0)
rows = S.generate_torch(3, device="cuda")
host = rows.cpu().pin_memory()
del rows
grid = S.grid_for(cfg)
acc = G.SufficientStatsAccumulator(grid, G.InterpScheme.Cubic, ctx=ctx)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    acc.reset()
    acc.add(host)
    t1 = time.perf_counter()
    st = acc.finalize()
    w = st.wty()
    t2 = time.perf_counter()
    print(f"add {1e3 * (t1 - t0):.2f} ms  finalize+wty {1e3 * (t2 - t1):.2f} ms  total {1e3 * (t2 - t0):.2f} ms  "
          f"(copy floor at 55.5 GB/s: {host.numel() * 4 / 55.5e9 * 1e3:.1f} ms)")

# copy-only reference: the same host chunks (2^24 rows) into two device slots, back to back
CH = 1 << 24
slots = [torch.empty((CH, host.shape[1]), dtype=host.dtype, device="cuda") for _ in range(2)]
cs = torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(cs):
        for k, a0 in enumerate(range(0, host.shape[0], CH)):
            a1 = min(host.shape[0], a0 + CH)
            slots[k & 1][: a1 - a0].copy_(host[a0:a1], non_blocking=True)
    cs.synchronize()
    t1 = time.perf_counter()
    print(f"copy only {1e3 * (t1 - t0):.2f} ms ({host.numel() * 4 / (t1 - t0) / 1e9:.1f} GB/s)")
