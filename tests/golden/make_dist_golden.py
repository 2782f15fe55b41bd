"""Generate tests/golden/dist_shards.npz ON A GPU BOX: the library's own reduce buffers
[stencil | W^T y | probe images | yty | n] and per-cell pattern bytes for two row shards of one
stream (probe streams positioned by enable_probes(first_row)) and for the single pass over all
rows.  tests/test_dist_gloo.py all-reduces the shard buffers with gloo through
distributed.allreduce_stats and must reproduce the single-pass buffers.

    python tests/golden/make_dist_golden.py   (needs libgsgpc + a CUDA device)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import paper_2101_11751_b200 as G  # noqa: E402
from paper_2101_11751_b200 import distributed as D  # noqa: E402


def data():
    rng = np.random.default_rng(11)
    x = rng.random((20000, 2))
    x[:400, 0] = np.round(x[:400, 0] * 12) / 12  # rows on grid lines: zero-weight patterns
    y = np.sin(5 * x[:, 0]) + 0.1 * rng.standard_normal(20000)
    return x, y


def buffers(g, x, y, first_row, probes=3, seed=5):
    acc = G.SufficientStatsAccumulator(g)
    acc.enable_probes(probes, seed=seed, first_row=first_row)
    acc.add(x, y)
    st = acc.finalize()
    return (D.stats_buffer_tensor(st).cpu().numpy().copy(), D.stats_pattern_tensor(st).cpu().numpy().copy(),
            st.n_offsets())


def main():
    x, y = data()
    g = G.fit_grid_to_data(np.zeros(2), np.ones(2), (17, 15))
    cut = 9001
    b0, p0, s_min = buffers(g, x[:cut], y[:cut], 0)
    b1, p1, _ = buffers(g, x[cut:], y[cut:], cut)
    bf, pf, _ = buffers(g, x, y, 0)
    np.savez_compressed(os.path.join(HERE, "dist_shards.npz"), x=x, y=y, cut=cut, sizes=np.array([17, 15]),
                        s_min=s_min, probes=3, seed=5, buf0=b0, buf1=b1, pat0=p0, pat1=p1, buf_full=bf,
                        pat_full=pf, version=G.version())
    print("wrote dist_shards.npz", b0.shape, p0.shape)


if __name__ == "__main__":
    main()
