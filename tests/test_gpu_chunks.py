"""Batches larger than one internal chunk (the reference's add() has no chunks: every row of
a call is one sequential pass, interp.cpp:188-200 / 244-263).  Host rows are staged in
equal chunks of ≤ 2^23 rows (copy of chunk k+1 overlapping the binning + moments of chunk
k); device rows are processed in chunks of ≤ 2^27.  The statistics must not depend on where
the chunk boundaries fall, the out-of-grid error must name the first bad row of the whole
call, and a failing call must leave the accumulator as it was."""
import numpy as np
import pytest

import paper_2101_11751_b200 as G

pytestmark = pytest.mark.gpu


def _rows(n, d, seed):
    import torch

    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.rand((n, d), generator=g, device="cuda", dtype=torch.float32) * 0.9 + 0.05
    y = torch.sin(3 * x).sum(dim=1) + 0.1 * torch.randn(n, generator=g, device="cuda", dtype=torch.float32)
    return x, y


def _same(a, b, tol=1e-11):
    assert a.n() == b.n()
    assert abs(a.yty() - b.yty()) <= 1e-12 * b.yty()
    np.testing.assert_allclose(a.wty(), b.wty(), rtol=tol, atol=tol * np.abs(b.wty()).max())
    va, oa = a.stencil()
    vb, ob = b.stencil()
    assert np.array_equal(oa, ob)
    np.testing.assert_allclose(va, vb, rtol=tol, atol=tol * np.abs(vb[0]).max())


def test_host_rows_over_several_staging_chunks():
    n = (1 << 23) + 54321  # two host chunks
    x, y = _rows(n, 2, 11)
    g = G.fit_grid_to_data([0.0, 0.0], [1.0, 1.0], [64, 48])
    dev = G.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
    xh, yh = x.cpu().pin_memory(), y.cpu().pin_memory()
    host = G.sufficient_stats(g, G.InterpScheme.Cubic, xh, yh)
    _same(host, dev)
    # pageable numpy rows take the same path
    _same(G.sufficient_stats(g, G.InterpScheme.Cubic, x.cpu().numpy(), y.cpu().numpy()), dev)


def test_host_error_in_last_chunk_rolls_back():
    n = (1 << 23) + 777
    x, y = _rows(n, 2, 12)
    xh, yh = x.cpu().numpy().copy(), y.cpu().numpy()
    bad = n - 5
    xh[bad, 1] = 1.5  # outside the grid, in the second staging chunk
    xh[bad + 2, 0] = -2.0
    g = G.fit_grid_to_data([0.0, 0.0], [1.0, 1.0], [40, 33])
    acc = G.SufficientStatsAccumulator(g, G.InterpScheme.Cubic)
    acc.add(xh[:1000], yh[:1000])
    before = acc.finalize()
    with pytest.raises(G.InvalidArgument) as e:
        acc.add(xh, yh)
    # rows are numbered after the rows already added (gsgpc_stats_add)
    assert e.value.row == 1000 + bad + 1 and "outside grid" in str(e.value)
    _same(acc.finalize(), before, tol=0.0)


def test_device_rows_over_several_chunks_and_rollback():
    n = (1 << 27) + 4097  # two device chunks
    x, y = _rows(n, 3, 13)
    g = G.fit_grid_to_data([0.0, 0.0, 0.0], [1.0, 1.0, 1.0], [20, 18, 16])
    one = G.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
    acc = G.SufficientStatsAccumulator(g, G.InterpScheme.Cubic)
    s = 50_000_001  # boundaries elsewhere: 5e7 | 2^27 | rest
    acc.add(x[:s], y[:s])
    acc.add(x[s:], y[s:])
    _same(acc.finalize(), one)
    # a bad row past the first device chunk: reported by its row, nothing committed
    bad = (1 << 27) + 17
    x[bad, 2] = 3.0
    acc.reset()
    acc.add(x[:1000], y[:1000])
    before = acc.finalize()
    with pytest.raises(G.InvalidArgument) as e:
        acc.add(x, y)
    assert e.value.row == 1000 + bad + 1 and "outside grid" in str(e.value)
    _same(acc.finalize(), before, tol=0.0)


def test_chunk_pipeline_gives_bitwise_the_sequential_statistics():
    """GSGPC_CHUNK_PIPE=1 overlaps the binning of chunk k + 1 with the moments kernel of chunk k on
    two scratch sets; kernels and accumulation order are the sequential path's, so the
    statistics must be bit-identical (the knob is read once per process: two subprocesses)."""
    import hashlib
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, hashlib, numpy as np\n"
        f"sys.path.insert(0, {root!r})\n"
        "import torch, paper_2101_11751_b200 as G\n"
        "g = torch.Generator(device='cuda').manual_seed(5)\n"
        "for d, sizes in ((2, [64, 48]), (3, [20, 16, 12])):\n"
        "    x = torch.rand((700_000, d), generator=g, device='cuda', dtype=torch.float32) * 0.9 + 0.05\n"
        "    y = torch.sin(3 * x).sum(dim=1)\n"
        "    grid = G.fit_grid_to_data([0.0] * d, [1.0] * d, sizes)\n"
        "    st = G.sufficient_stats(grid, G.InterpScheme.Cubic, x, y)\n"
        "    h = hashlib.sha256(st.stencil()[0].tobytes() + st.wty().tobytes() + np.float64(st.yty()).tobytes())\n"
        "    print(d, st.n(), h.hexdigest())\n"
    )
    outs = []
    for pipe in ("0", "1"):
        env = dict(os.environ, GSGPC_CHUNK_PIPE=pipe, GSGPC_DEV_CHUNK_LOG2="16")  # 11 chunks
        res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        outs.append(res.stdout)
    assert outs[0] == outs[1] and outs[0].count("\n") == 2
    del hashlib
