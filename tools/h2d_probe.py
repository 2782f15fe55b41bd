"""Host→device copy bandwidth from pinned memory: one stream vs several (diagnostics)."""
import time

import torch

N = 1 << 28  # 256 Mi floats = 1 GiB
h = torch.empty(N, dtype=torch.float32).pin_memory()
d = torch.empty(N, dtype=torch.float32, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    part = N // ns
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
    print(f"streams={ns}: {N * 4 / el / 1e9:.1f} GB/s")
