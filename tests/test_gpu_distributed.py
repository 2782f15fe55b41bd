"""The multi-GPU combine path on one GPU: paper_2101_11751_b200.distributed.allreduce_stats
(the NCCL all-reduce `bench.py --gpus N` runs after each rank's precompute) under a
single-rank NCCL process group.  With one rank the sum is the identity, so the reduced
statistics must equal the unreduced ones bit for bit — which exercises the device view of
the reduce buffer, the in-place collective, mark_reduced and every accessor on reduced
statistics (n and yᵀy read back from the buffer tail).  The two-rank arithmetic of the
combine (merge() semantics) is covered on CPU by test_dist_gloo.py."""
import os
import socket

import numpy as np
import pytest

import paper_2101_11751_b200 as G
from test_gpu_parity import points

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_single_rank_nccl_allreduce_is_identity():
    import torch
    import torch.distributed as dist

    from paper_2101_11751_b200.distributed import allreduce_stats

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = G.fit_grid_to_data(np.zeros(3), np.ones(3), (11, 9, 8))
        x, y = points(3, 30000, 21)
        ref = G.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
        st = G.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
        ref_vals, ref_offs = ref.stencil()
        allreduce_stats(st)
        vals, offs = st.stencil()
        assert np.array_equal(offs, ref_offs)
        # the binning order is not deterministic, so compare to rounding, not bits
        np.testing.assert_allclose(vals, ref_vals, rtol=1e-12, atol=1e-12 * np.abs(ref_vals).max())
        np.testing.assert_allclose(st.wty(), ref.wty(), rtol=1e-12, atol=1e-12 * np.abs(ref.wty()).max())
        assert st.n() == ref.n() == 30000
        assert abs(st.yty() - ref.yty()) <= 1e-12 * ref.yty()
        # a solve on the reduced statistics (every rank holds the merged statistics)
        spec = G.KernelSpec(G.Hyperparams(3.0, [0.3, 0.3, 0.4], 1.0))
        kg = G.ToeplitzOperator(g, spec)
        m1 = G.posterior_mean_gsgp(st, kg, spec, G.InterpScheme.Cubic, 3.0, 1e-8, 2000)
        m0 = G.posterior_mean_gsgp(ref, kg, spec, G.InterpScheme.Cubic, 3.0, 1e-8, 2000)
        assert np.abs(m1.mean_coeffs - m0.mean_coeffs).max() <= 1e-6 * np.abs(m0.mean_coeffs).max()
        # reduced statistics refuse further rows (a new accumulator pass starts from reset)
        with pytest.raises(G.InvalidArgument, match="all-reduced"):
            acc = G.SufficientStatsAccumulator(g)
            acc.add(x[:10], y[:10])
            s2 = acc.finalize()
            allreduce_stats(s2)
            acc.add(x[:10], y[:10])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("route", ["ski", "sym"])
def test_probe_shards_combine_to_the_full_slq(route):
    """SLQ probes split over ranks.  Each probe's Lanczos run is independent of the
    others in its batch, so shards combined (Σ per-probe estimates / P + shift) reproduce the
    single-call log-likelihood to rounding."""
    from paper_2101_11751_b200.distributed import combine_loglik, probe_shard

    g = G.fit_grid_to_data(np.zeros(3), np.ones(3), (10, 9, 8))
    x, y = points(3, 8000, 5)
    spec = G.KernelSpec(G.Hyperparams(0.1, [0.2, 0.25, 0.3], 1.0))
    kg = G.ToeplitzOperator(g, spec)
    if route == "ski":
        acc = G.SufficientStatsAccumulator(g)
        acc.enable_probes(10, seed=3)
        acc.add(x, y)
        st = acc.finalize()
        base = G.LoglikOptions(solve_tol=1e-9, probes=10, slq=G.SlqOptions(max_depth=30, quad_tol=0.0), seed=3,
                               maxiter=5000, route=G.LogdetRoute.SkiOperator)
    else:
        st = G.sufficient_stats(g, G.InterpScheme.Cubic, x, y)
        base = G.LoglikOptions(solve_tol=1e-9, probes=10, slq=G.SlqOptions(max_depth=30, quad_tol=0.0), seed=3,
                               maxiter=5000, route=G.LogdetRoute.SymmetricGrid)
    full = G.log_likelihood_gsgp(st, kg, 0.1, base)
    import dataclasses
    parts = []
    for r in range(3):
        b, e = probe_shard(10, 3, r)
        parts.append(G.log_likelihood_gsgp(st, kg, 0.1, dataclasses.replace(base, probe_begin=b, probe_end=e)))
    assert [p.slq_count for p in parts] == [4, 4, 2]
    comb = combine_loglik(parts, full.quad_term, full.const_term)
    assert comb.slq_count == full.slq_count == 10
    assert abs(comb.logdet_term - full.logdet_term) <= 1e-12 * abs(full.logdet_term)
    assert abs(comb.loglik - full.loglik) <= 1e-12 * abs(full.loglik)


def test_sharded_loglik_single_rank_group():
    import torch
    import torch.distributed as dist

    from paper_2101_11751_b200.distributed import log_likelihood_gsgp_sharded

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = G.fit_grid_to_data(np.zeros(2), np.ones(2), (16, 14))
        x, y = points(2, 6000, 9)
        acc = G.SufficientStatsAccumulator(g)
        acc.enable_probes(6, seed=1)
        acc.add(x, y)
        st = acc.finalize()
        kg = G.ToeplitzOperator(g, G.KernelSpec(G.Hyperparams(0.1, [0.2, 0.25], 1.0)))
        opts = G.LoglikOptions(solve_tol=1e-9, probes=6, slq=G.SlqOptions(max_depth=20, quad_tol=0.0), seed=1,
                               maxiter=5000)
        a = G.log_likelihood_gsgp(st, kg, 0.1, opts)
        b = log_likelihood_gsgp_sharded(st, kg, 0.1, opts)
        assert abs(a.loglik - b.loglik) <= 1e-12 * abs(a.loglik)
        assert b.probes_used == a.probes_used == 6
    finally:
        dist.destroy_process_group()
