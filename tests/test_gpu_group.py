"""The in-process multi-GPU entry point (gsgpc_group_*: SURVEY §8(b) gsgpc_ctx_create(device_ids[],
ngpu), §8(e) row sharding + one all-reduce with merge() semantics, interp.cpp:202-210).

One GPU per test box: a group that lists device 0 several times runs every shard on it and
exchanges through peer copies (the NCCL path needs distinct devices; it is taken when
available and the test below checks it whenever the box has ≥ 2 GPUs).  The merged statistics
must equal the oracle's on all rows, every device's copy must be identical, probe images must
equal the one-device streams (each shard starts its streams at its first row), and an
out-of-grid row in a later shard must be reported at its row in the whole batch."""
import numpy as np
import pytest

import oracle as O
import paper_2101_11751_b200 as G
from helpers import csr_to_half_stencil, rel_err

pytestmark = pytest.mark.gpu


def ogrid(g):
    return O.Grid([g.min(k) for k in range(g.dim())], [g.max(k) for k in range(g.dim())],
                  [g.size(k) for k in range(g.dim())])


def _case(n=90_000, d=3, seed=5):
    rng = np.random.default_rng(seed)
    x = rng.random((n, d))
    y = np.sin(5 * x).sum(axis=1) + 0.1 * rng.standard_normal(n)
    g = G.fit_grid_to_data(np.zeros(d), np.ones(d), (14, 12, 10)[:d])
    return g, x, y


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_group_stats_match_oracle(devices):
    g, x, y = _case()
    grp = G.DeviceGroup(devices)
    assert len(grp) == len(devices) and not grp.uses_nccl
    sts = grp.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
    os_ = O.sufficient_stats(ogrid(g), x, y, scheme=1, nthreads=8)
    rp, col, val, owty = os_.csr()
    ref = csr_to_half_stencil(rp, col, val, (14, 12, 10), 4)
    first = None
    for st in sts:
        vals, _ = st.stencil()
        assert np.abs(vals - ref).max() <= 1e-10 * np.abs(ref[0]).max()
        assert rel_err(st.wty(), owty) <= 1e-10
        assert st.n() == os_.n and abs(st.yty() - os_.yty) <= 1e-12 * os_.yty
        grp_rp, grp_col, _ = st.csr()
        assert np.array_equal(grp_rp, rp) and np.array_equal(grp_col, col)  # merged structure
        if first is None:
            first = (vals, st.wty())
        else:  # every device holds the same merged statistics
            assert np.array_equal(vals, first[0]) and np.array_equal(st.wty(), first[1])


def test_group_probe_images_equal_one_device_streams():
    g, x, y = _case(n=40_000, d=2)
    grp = G.DeviceGroup([0, 0])
    sts = grp.sufficient_stats(g, G.InterpScheme.Cubic, x, y, probes=5, seed=9)
    acc = G.SufficientStatsAccumulator(g)
    acc.enable_probes(5, seed=9)
    acc.add(x, y)
    one = acc.finalize()
    assert rel_err(sts[0].probe_images(), one.probe_images()) <= 1e-12
    assert rel_err(sts[1].probe_images(), one.probe_images()) <= 1e-12


def test_group_out_of_grid_row_is_global():
    g, x, y = _case(n=30_000)
    x[20_001] = 5.0  # in the second of three shards
    x[25_000] = -1.0
    grp = G.DeviceGroup([0, 0, 0])
    with pytest.raises(G.InvalidArgument) as ei:
        grp.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
    assert ei.value.row == 20_002 and "stream row 20002" in str(ei.value)


def test_group_solve_on_merged_stats():
    """The replicated solve on a device's merged statistics equals the one-device solve."""
    g, x, y = _case(n=60_000)
    spec = G.KernelSpec(G.Hyperparams(1.0, [0.12, 0.12, 0.12], 1.0))  # well conditioned
    grp = G.DeviceGroup([0, 0])
    sts = grp.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
    one = G.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
    kg = G.ToeplitzOperator(g, spec, ctx=grp.context(1))
    m1 = G.posterior_mean_gsgp(sts[1], kg, spec, G.InterpScheme.Cubic, 1.0, 1e-8, 5000)
    m0 = G.posterior_mean_gsgp(one, G.ToeplitzOperator(g, spec), spec, G.InterpScheme.Cubic, 1.0, 1e-8, 5000)
    # the merged statistics equal the one-device ones to rounding (summation order), which moves
    # CG iteration counts on this moderately conditioned system by a few
    assert abs(m1.solve_iterations - m0.solve_iterations) <= max(2, m0.solve_iterations // 20)
    assert rel_err(m1.mean_coeffs, m0.mean_coeffs) <= 1e-6


def test_group_nccl_when_distinct_devices():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    g, x, y = _case()
    grp = G.DeviceGroup([0, 1])
    sts = grp.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
    one = G.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
    for st in sts:
        assert rel_err(st.stencil()[0], one.stencil()[0]) <= 1e-12
        assert st.n() == one.n()
