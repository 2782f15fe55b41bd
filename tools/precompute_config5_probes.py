import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2101_11751_b200 as G
from paper_2101_11751_b200 import synthetic as S
cfg = S.CONFIGS[5]
ctx = G.Context(0)
rows = S.generate_torch(5, device="cuda")
grid = S.grid_for(cfg)
for rep in range(2):
    acc = G.SufficientStatsAccumulator(grid, G.InterpScheme.Cubic, ctx=ctx)
    acc.enable_probes(30, seed=0)
    acc.add(rows)
    st = acc.finalize()
    torch.cuda.synchronize()
print("ok")
