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


def test_persistent_cg_after_solves_with_other_shared_memory_sizes():
    """The persistent CG kernel's function attributes (dynamic shared memory, carveout) are per
    kernel, not per launch: a solve on a large grid must still launch after solves of the same
    dimension on smaller grids changed them (regression: 'too many blocks in cooperative launch'
    when the cached grid met another launch's carveout), with bitwise the same result."""
    ctx = G.Context(0)
    rng = np.random.default_rng(9)
    spec = G.KernelSpec(G.Hyperparams(0.3, [0.05, 0.05], 1.0))

    def solve(sizes, n):
        x = np.random.default_rng(sizes[0]).random((n, 2))
        y = np.sin(3.0 * x.sum(axis=1))
        g = G.fit_grid_to_data(np.zeros(2), np.ones(2), sizes, G.InterpScheme.Cubic)
        st = G.sufficient_stats(g, G.InterpScheme.Cubic, x, y, ctx=ctx)
        kg = G.ToeplitzOperator(g, spec, ctx=ctx)
        r0 = -kg.apply(st.wty()) / 0.09
        res = G.factorized_cg_grid_rhs(kg, st, r0, 0.3, G.GridRhsTolerance(eps_abs=1e-30), 12)
        return res.xhat_d.copy(), res.residual_trace.copy()

    first = solve((256, 256), 400_000)
    for sizes in ((20, 17), (64, 48), (700, 30), (9, 300)):
        solve(sizes, 20_000)
    again = solve((256, 256), 400_000)
    assert np.array_equal(first[0].view(np.uint64), again[0].view(np.uint64))
    assert np.array_equal(first[1].view(np.uint64), again[1].view(np.uint64))
    del rng
