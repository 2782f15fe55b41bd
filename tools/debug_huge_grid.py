import sys, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import paper_2101_11751_b200 as G
sizes=(3000,3000)
g=G.fit_grid_to_data(np.zeros(2),np.ones(2),sizes,G.InterpScheme.Cubic)
rng=np.random.default_rng(23); x=rng.random((200000,2)); y=np.cos(4*x).sum(axis=1)
ctx=G.Context(0)
gs=G.sufficient_stats(g,G.InterpScheme.Cubic,x,y,ctx=ctx)
print('n',gs.n(), 'launches', ctx.launch_count)
