"""Multi-rank combination of the statistics on CPU (gloo, world_size 2).

Each rank computes the statistics of its own shard of rows, packs them in the device
reduce-buffer layout [half stencil (S_min·m) | W^T y (m) | yty | n] that
gsgpc_stats_reduce_buffer exposes, and the ranks sum them with all_reduce — the
reference's SufficientStatsAccumulator::merge (interp.cpp:202-210).  The result must equal
the statistics of all rows (the same code path the NCCL run takes on the GPU box,
paper_2101_11751_b200/distributed.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from helpers import csr_to_half_stencil


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    rng = np.random.default_rng(11)
    x = rng.random((20000, 2))
    y = np.sin(5 * x[:, 0]) + 0.1 * rng.standard_normal(20000)
    g = O.fit_grid_to_data([0, 0], [1, 1], [17, 15])
    return g, x, y


def _pack(st, sizes):
    rp, col, val, wty = st.csr()
    half = csr_to_half_stencil(rp, col, val, sizes, 4)
    return np.concatenate([half.reshape(-1), wty, [st.yty, float(st.n)]])


def _sparse():
    # ~0.5 rows per cell: every shard touches a different set of W^T W pairs
    rng = np.random.default_rng(12)
    x = rng.random((1500, 2))
    x[:300, 0] = np.round(x[:300, 0] * 40) / 40  # some rows on grid lines (t = 0 in dimension 0)
    y = rng.standard_normal(1500)
    g = O.fit_grid_to_data([0, 0], [1, 1], [60, 50])
    return g, x, y


def _structure(st, sizes):
    """The touched-pair mask of W^T W in half-stencil layout, one byte per entry — what
    gsgpc_stats_pattern_buffer's per-cell patterns encode and ranks combine by MAX (= OR)."""
    rp, col, _, _ = st.csr()
    mask = csr_to_half_stencil(rp, col, np.ones(len(col)), sizes, 4)
    return mask.reshape(-1).astype(np.uint8)


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, x, y = _data()
    lo, hi = rank * x.shape[0] // world, (rank + 1) * x.shape[0] // world
    st = O.sufficient_stats(g, x[lo:hi], y[lo:hi])
    t = torch.from_numpy(_pack(st, [17, 15]))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    np.save(f"{out_path}.{rank}.npy", t.numpy())
    gs, xs, ys = _sparse()
    lo, hi = rank * xs.shape[0] // world, (rank + 1) * xs.shape[0] // world
    mk = torch.from_numpy(_structure(O.sufficient_stats(gs, xs[lo:hi], ys[lo:hi]), [60, 50]))
    dist.all_reduce(mk, op=dist.ReduceOp.MAX)
    np.save(f"{out_path}.mask.{rank}.npy", mk.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_allreduce_equals_merge(tmp_path):
    world = 2
    port = _free_port()
    out = str(tmp_path / "buf")
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
    g, x, y = _data()
    full = _pack(O.sufficient_stats(g, x, y), [17, 15])
    for r in range(world):
        got = np.load(f"{out}.{r}.npy")
        assert got[-1] == full[-1]  # n exact
        np.testing.assert_allclose(got, full, rtol=1e-12, atol=1e-12 * np.abs(full).max())
    gs, xs, ys = _sparse()
    full_mask = _structure(O.sufficient_stats(gs, xs, ys), [60, 50])
    for r in range(world):
        got = np.load(f"{out}.mask.{r}.npy")
        assert np.array_equal(got, full_mask)  # structure of the union = OR of the shards'


GOLD = os.path.join(os.path.dirname(__file__), "golden", "dist_shards.npz")


class _LibraryBuffers:
    """A rank's statistics as libgsgpc wrote them on a B200 (tests/golden/make_dist_golden.py):
    the reduce buffer [stencil | W^T y | probe images | yty | n] and the per-cell pattern bytes,
    in host tensors, with the interface distributed.allreduce_stats drives."""

    class _Ctx:
        def synchronize(self):
            pass

    def __init__(self, buf, pat):
        self.buf = torch.from_numpy(buf.copy())
        self.pat = torch.from_numpy(pat.copy())
        self.context = self._Ctx()
        self.reduced = False

    def reduce_tensor(self):
        return self.buf

    def pattern_tensor(self):
        return self.pat

    def mark_reduced(self):
        self.reduced = True


def _lib_worker(rank, world, port, out_path):
    from paper_2101_11751_b200.distributed import allreduce_stats

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z = np.load(GOLD)
    st = _LibraryBuffers(z[f"buf{rank}"], z[f"pat{rank}"])
    allreduce_stats(st)
    assert st.reduced
    np.save(f"{out_path}.{rank}.npy", st.buf.numpy())
    np.save(f"{out_path}.pat.{rank}.npy", st.pat.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(not os.path.exists(GOLD), reason="tests/golden/dist_shards.npz not generated")
def test_allreduce_stats_on_library_buffers(tmp_path):
    """distributed.allreduce_stats (the function the NCCL ranks call) over gloo, on the library's
    own shard buffers: two row shards of one stream, their probe streams positioned by
    enable_probes(first_row).  The all-reduced buffers equal the library's single pass over all
    rows (values to 1e-12, n exact, structure bytes identical), and the stencil / W^T y part
    equals the oracle's merge() of the same rows."""
    world = 2
    port = _free_port()
    out = str(tmp_path / "lib")
    mp.start_processes(_lib_worker, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
    z = np.load(GOLD)
    full, pfull = z["buf_full"], z["pat_full"]
    sizes = [int(v) for v in z["sizes"]]
    m = int(np.prod(sizes))
    s_min = int(z["s_min"])
    for r in range(world):
        got = np.load(f"{out}.{r}.npy")
        assert got[-1] == full[-1] == z["x"].shape[0]  # n exact
        np.testing.assert_allclose(got, full, rtol=1e-12, atol=1e-12 * np.abs(full).max())
        assert np.array_equal(np.load(f"{out}.pat.{r}.npy"), pfull)
    # against the oracle's statistics of all rows (stencil, W^T y, yty)
    g = O.fit_grid_to_data([0, 0], [1, 1], sizes)
    ost = O.sufficient_stats(g, z["x"], z["y"])
    rp, col, val, wty = ost.csr()
    ref = csr_to_half_stencil(rp, col, val, sizes, 4).reshape(-1)
    got = np.load(f"{out}.0.npy")
    assert np.abs(got[: s_min * m] - ref).max() <= 1e-10 * np.abs(ref).max()
    assert np.abs(got[s_min * m: s_min * m + m] - wty).max() <= 1e-10 * np.abs(wty).max()
    assert abs(got[-2] - ost.yty) <= 1e-12 * ost.yty
    # probe images of the shards sum to the single-stream images of rademacher_probe
    P = int(z["probes"])
    img = got[s_min * m + m: s_min * m + m + P * m].reshape(P, m)
    for p in range(P):
        v = O.rademacher_probe(z["x"].shape[0], int(z["seed"]), p)
        ri = O.wt_apply(g, z["x"], v)
        assert np.abs(img[p] - ri).max() <= 1e-10 * np.abs(ri).max()


def test_probe_shards_cover_the_probe_set():
    from paper_2101_11751_b200.distributed import probe_shard

    for P in (1, 7, 30, 64):
        for world in (1, 2, 3, 8):
            shards = [probe_shard(P, world, r) for r in range(world)]
            covered = [p for b, e in shards for p in range(b, e)]
            assert covered == list(range(P))
            assert max(e - b for b, e in shards) == -(-P // world)


def test_combine_loglik_arithmetic():
    from paper_2101_11751_b200.distributed import combine_loglik
    from paper_2101_11751_b200.gsgp import LoglikResult

    parts = [LoglikResult(slq_sum=10.0, slq_count=4, logdet_shift=-2.0, probes_used=4, max_depth_used=5),
             LoglikResult(slq_sum=8.0, slq_count=4, logdet_shift=-2.0, probes_used=4, max_depth_used=7),
             LoglikResult(slq_sum=3.0, slq_count=2, logdet_shift=-2.0, probes_used=2, max_depth_used=6)]
    r = combine_loglik(parts, quad_term=5.0, const_term=1.0)
    assert r.logdet_term == 21.0 / 10 - 2.0
    assert r.loglik == -0.5 * (r.logdet_term + 5.0 + 1.0)
    assert r.probes_used == 10 and r.max_depth_used == 7
