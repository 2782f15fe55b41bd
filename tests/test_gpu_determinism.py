"""Bitwise reproducibility of the precompute (the reference's add() is sequential in stream
order, interp.cpp:188-200, so it returns the same statistics on every run): two passes over the
same rows give identical W^T W stencil, W^T y, yᵀy and probe-image bytes — deterministic bucket
and cell ranks in the binning (det_slot), fixed per-warp row ranges in K1, one add per cell
(split records), fixed-order reductions.  Covers every K1 kernel: d = 3 cubic (DMMA), d = 2 cubic
(DMMA), the lane kernel (d = 1, linear), the probe moments (DMMA and lane), and both slice
scatters (direct: long runs per cell; staged: config 4's 1024-cell buckets)."""
import numpy as np
import pytest

import paper_2101_11751_b200 as G

pytestmark = pytest.mark.gpu


def twice(g, scheme, rows, probes=0, seed=0):
    out = []
    for _ in range(2):
        acc = G.SufficientStatsAccumulator(g, scheme)
        if probes:
            acc.enable_probes(probes, seed=seed)
        acc.add(rows)
        st = acc.finalize()
        out.append((st.stencil()[0], st.wty(), st.yty(), st.probe_images() if probes else None))
    return out


def assert_same(a, b):
    assert np.array_equal(a[0].view(np.uint64), b[0].view(np.uint64))
    assert np.array_equal(a[1].view(np.uint64), b[1].view(np.uint64))
    assert a[2] == b[2]
    if a[3] is not None:
        assert np.array_equal(a[3].view(np.uint64), b[3].view(np.uint64))


@pytest.mark.parametrize("cfg_id,n,probes", [(3, None, 0), (5, None, 30), (4, 100_000_000, 0), (2, None, 0),
                                             (1, None, 0), (5, 3_000_000, 5)])
def test_precompute_bitwise_reproducible(cfg_id, n, probes):
    import torch

    from paper_2101_11751_b200 import synthetic as S

    cfg = S.CONFIGS[cfg_id]
    rows = S.generate_torch(cfg_id, n, device="cuda")
    a, b = twice(S.grid_for(cfg), G.InterpScheme.Cubic, rows, probes)
    del rows
    torch.cuda.empty_cache()
    assert_same(a, b)


@pytest.mark.parametrize("scheme", [G.InterpScheme.Linear, G.InterpScheme.Cubic])
def test_lane_kernels_bitwise_reproducible(scheme):
    """d = 3 linear (lane kernel) and d = 1 with probes (lane probe kernel)."""
    rng = np.random.default_rng(3)
    x = rng.random((2_000_000, 3))
    y = rng.standard_normal(2_000_000)
    g = G.fit_grid_to_data(np.zeros(3), np.ones(3), (30, 20, 10), scheme)
    a, b = twice(g, scheme, np.column_stack([x, y]))
    assert_same(a, b)
    g1 = G.fit_grid_to_data([0.0], [1.0], [200], scheme)
    a, b = twice(g1, scheme, np.column_stack([x[:, :1], y]), probes=7, seed=3)
    assert_same(a, b)


def test_posterior_mean_reproducible_end_to_end():
    """Precompute + posterior_mean_gsgp twice on BASELINE config 1 (1e6 rows, ~800 iterations of
    an ill-conditioned system): same iteration count, bitwise-identical coefficients."""
    from paper_2101_11751_b200 import synthetic as S

    cfg = S.CONFIGS[1]
    g = S.grid_for(cfg)
    spec = S.kernel_for(cfg)
    x, y = S.generate(1)
    res = []
    for _ in range(2):
        st = G.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
        kg = G.ToeplitzOperator(g, spec)
        res.append(G.posterior_mean_gsgp(st, kg, spec, G.InterpScheme.Cubic, cfg.noise_std, cfg.tol, 5000))
    assert res[0].solve_iterations == res[1].solve_iterations
    assert np.array_equal(res[0].mean_coeffs, res[1].mean_coeffs)
