"""Two contexts on one device, driven from two host threads at once (the reference's
ToeplitzOperator/SufficientStats are safe for concurrent use, grid.hpp:55-57): every table a
kernel reads (stencil offsets, weight-polynomial coefficients, persistent-grid attributes) is
per launch or per device, so a d = 2 cubic, a d = 3 cubic and a d = 3 linear precompute + solve
running concurrently give bitwise the results each gives alone (the precompute and the
persistent CG are bitwise reproducible, tests/test_gpu_determinism.py)."""
import threading

import numpy as np
import pytest

import paper_2101_11751_b200 as G

pytestmark = pytest.mark.gpu


def _case(kind):
    rng = np.random.default_rng({"d2": 1, "d3": 2, "d3lin": 3}[kind])
    if kind == "d2":
        d, sizes, scheme, n = 2, (96, 80), G.InterpScheme.Cubic, 1_500_000
    elif kind == "d3":
        d, sizes, scheme, n = 3, (24, 20, 12), G.InterpScheme.Cubic, 1_500_000
    else:
        d, sizes, scheme, n = 3, (30, 18, 10), G.InterpScheme.Linear, 1_500_000
    x = rng.random((n, d))
    y = np.sin(3.0 * x.sum(axis=1)) + 0.1 * rng.standard_normal(n)
    g = G.fit_grid_to_data(np.zeros(d), np.ones(d), sizes, scheme)
    spec = G.KernelSpec(G.Hyperparams(0.3, [0.15] * d, 1.0))
    return g, scheme, spec, x, y


def _run(kind, ctx, reps=3):
    g, scheme, spec, x, y = _case(kind)
    out = None
    for _ in range(reps):
        st = G.sufficient_stats(g, scheme, x, y, ctx=ctx)
        kg = G.ToeplitzOperator(g, spec, ctx=ctx)
        model = G.posterior_mean_gsgp(st, kg, spec, scheme, 0.3, 1e-6, 20000)
        res = (st.stencil()[0].copy(), st.wty().copy(), model.mean_coeffs.copy(), model.solve_iterations)
        if out is None:
            out = res
        else:  # every repetition inside the concurrent run agrees with the first
            assert_same(out, res)
    return out


def assert_same(a, b):
    assert np.array_equal(a[0].view(np.uint64), b[0].view(np.uint64))
    assert np.array_equal(a[1].view(np.uint64), b[1].view(np.uint64))
    assert np.array_equal(a[2].view(np.uint64), b[2].view(np.uint64))
    assert a[3] == b[3]


def test_two_contexts_one_device_concurrently():
    kinds = ["d2", "d3", "d3lin"]
    alone = {k: _run(k, G.Context(0), reps=1) for k in kinds}
    got, errs = {}, []

    def worker(k):
        try:
            got[k] = _run(k, G.Context(0))
        except Exception as e:  # noqa: BLE001
            errs.append((k, e))

    ths = [threading.Thread(target=worker, args=(k,)) for k in kinds]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs, errs
    for k in kinds:
        assert_same(alone[k], got[k])


def test_foreign_device_pointer_rejected():
    """A device array on another GPU than the context's is an INVALID_ARGUMENT, not a silent
    dereference of a foreign address (only checkable with two GPUs)."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    g = G.fit_grid_to_data([0.0], [1.0], [50], G.InterpScheme.Cubic)
    rows = torch.rand(1000, 2, dtype=torch.float64, device="cuda:1")
    with pytest.raises(G.InvalidArgument, match="device"):
        G.sufficient_stats(g, G.InterpScheme.Cubic, rows[:, :1].contiguous(), rows[:, 1].contiguous(),
                           ctx=G.Context(0))
