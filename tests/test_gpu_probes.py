"""Probe streams through the precompute on the GPU: substream generation (slabs split into
1,048,320-draw substreams started by the GF(2) jump-ahead) and shard offsets
(enable_probes(first_row)), against the oracle's sequential rademacher_probe (gp.cpp:16-25)."""
import numpy as np
import pytest

import oracle as O
import paper_2101_11751_b200 as G
from helpers import rel_err

pytestmark = pytest.mark.gpu


def ogrid(g):
    return O.Grid([g.min(k) for k in range(g.dim())], [g.max(k) for k in range(g.dim())],
                  [g.size(k) for k in range(g.dim())])


def case(n, seed=3):
    rng = np.random.default_rng(seed)
    x = rng.random((n, 2))
    y = np.sin(6 * x[:, 0]) + 0.1 * rng.standard_normal(n)
    g = G.fit_grid_to_data(np.zeros(2), np.ones(2), (16, 14))
    return g, x, y


def oracle_images(g, x, seed, probes):
    og = ogrid(g)
    return np.array([O.wt_apply(og, x, O.rademacher_probe(x.shape[0], seed, p)) for p in probes])


def test_substream_probe_images_match_oracle():
    """2.6e6 rows in two batches: the first batch spans 2 substreams, the second 2 more,
    continuing from the first batch's end state."""
    n = 2_600_000
    g, x, y = case(n)
    P = 4
    acc = G.SufficientStatsAccumulator(g)
    acc.enable_probes(P, seed=11)
    acc.add(x[:1_500_000], y[:1_500_000])
    acc.add(x[1_500_000:], y[1_500_000:])
    img = acc.finalize().probe_images()
    ref = oracle_images(g, x, 11, range(P))
    for p in range(P):
        assert rel_err(img[p], ref[p]) <= 1e-10, p


def test_sharded_probe_streams_sum_to_single_pass():
    """Three shards of one stream (first_row = global offset of each shard's first row) merge to
    the single-pass images; merging shards that are not adjacent is refused."""
    n = 300_000
    g, x, y = case(n, seed=4)
    P = 3
    cuts = [0, 70_001, 190_000, n]
    shards = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        acc = G.SufficientStatsAccumulator(g)
        acc.enable_probes(P, seed=2, first_row=a)
        acc.add(x[a:b], y[a:b])
        shards.append(acc)
    bad = G.SufficientStatsAccumulator(g)
    bad.enable_probes(P, seed=2, first_row=cuts[2])
    bad.add(x[cuts[2]:], y[cuts[2]:])
    with pytest.raises(G.InvalidArgument):
        shards[0].merge(bad)  # rows [0, 70001) and [190000, n) are not adjacent
    shards[1].merge(shards[2])  # [70001, n)
    shards[0].merge(shards[1])  # [0, n)
    img = shards[0].finalize().probe_images()
    single = G.SufficientStatsAccumulator(g)
    single.enable_probes(P, seed=2)
    single.add(x, y)
    ref1 = single.finalize().probe_images()
    ref = oracle_images(g, x, 2, range(P))
    for p in range(P):
        assert rel_err(img[p], ref[p]) <= 1e-10, p
        assert rel_err(img[p], ref1[p]) <= 1e-12, p
    # the merged accumulator continues the stream after its last row
    more_x, more_y = case(50_000, seed=9)[1:]
    shards[0].add(more_x, more_y)
    single.add(more_x, more_y)
    a2 = shards[0].finalize().probe_images()
    b2 = single.finalize().probe_images()
    assert rel_err(a2, b2) <= 1e-12


def test_config5_probe_streams_on_substreams():
    """BASELINE config 5's 30 probes on a 2.2e6-row prefix (three substreams per probe):
    probes 0, 17 and 29 against the oracle's sequential streams."""
    import torch

    from paper_2101_11751_b200 import synthetic as S

    cfg = S.CONFIGS[5]
    g = S.grid_for(cfg)
    rows = S.generate_torch(5, 2_200_000, device="cuda")
    acc = G.SufficientStatsAccumulator(g)
    acc.enable_probes(30, seed=0)
    acc.add(rows)
    img = acc.finalize().probe_images()
    host = rows.cpu().numpy()
    del rows
    torch.cuda.empty_cache()
    ref = oracle_images(g, host[:, :3], 0, (0, 17, 29))
    for i, p in enumerate((0, 17, 29)):
        assert rel_err(img[p], ref[i]) <= 1e-10, p
