"""Multi-GPU combination of per-rank sufficient statistics.

Each rank (one process per GPU) runs the precompute on its own shard of rows; the partial
statistics are combined by an in-place sum all-reduce of the finalized device buffer
[stencil | W^T y | probe images | yty | n] — the reference's
SufficientStatsAccumulator::merge semantics (interp.cpp:202-210, elementwise sums),
carried over NCCL (NVLink / NVSwitch) by torch.distributed.  finalize() is linear in the
cell moments, so reducing finalized buffers equals finalizing reduced moments.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class _DevView:
    def __init__(self, ptr: int, count: int, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def stats_buffer_tensor(stats, device=None) -> torch.Tensor:
    """A torch view (no copy) of the stats' reduce buffer."""
    ptr, count = stats.reduce_buffer()
    dev = device if device is not None else torch.device("cuda", stats.context.device)
    return torch.as_tensor(_DevView(ptr, count), device=dev)


def stats_pattern_tensor(stats, device=None) -> torch.Tensor:
    """A torch view (no copy) of the stats' per-cell zero-weight pattern bytes (the W^T W
    structure, kept apart from the values); ranks combine them by MAX (= OR)."""
    ptr, count = stats.pattern_buffer()
    dev = device if device is not None else torch.device("cuda", stats.context.device)
    return torch.as_tensor(_DevView(ptr, count, "|u1"), device=dev)


def allreduce_stats(stats, group=None):
    """Sum the finalized statistics of every rank in place (all ranks end with the merged
    statistics) and mark the object reduced.

    `stats` exposes reduce_tensor() / pattern_tensor() (views of the library's device buffers
    for SufficientStats), context.synchronize() and mark_reduced(); the CPU tests hand in the
    same buffers, as the library wrote them on a B200, held in host tensors (gloo)."""
    buf = stats.reduce_tensor()
    pat = stats.pattern_tensor()
    stats.context.synchronize()
    work = dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group, async_op=True)
    dist.all_reduce(pat, op=dist.ReduceOp.MAX, group=group)
    work.wait()
    if buf.is_cuda:
        torch.cuda.current_stream(buf.device).synchronize()
    stats.mark_reduced()
    return stats


def probe_shard(probes: int, world: int, rank: int):
    """Contiguous ⌈P/G⌉ probe shard of rank `rank` (SLQ probes split over GPUs)."""
    per = -(-probes // world)
    b = min(probes, rank * per)
    return b, min(probes, b + per)


def combine_loglik(results, quad_term, const_term):
    """Combine per-shard LoglikResults (same statistics, disjoint probe shards): the log
    determinant is the mean of the per-probe estimates over all shards, plus the route's
    shift; the quadratic and constant terms are the same on every shard."""
    from .gsgp import LoglikResult

    total = sum(r.slq_sum for r in results)
    count = sum(r.slq_count for r in results)
    r0 = results[0]
    logdet = total / count + r0.logdet_shift if count > 0 else r0.logdet_term
    return LoglikResult(-0.5 * (logdet + quad_term + const_term), logdet, quad_term, const_term,
                        sum(r.probes_used for r in results), r0.solver_iterations, r0.logdet_route,
                        max(r.max_depth_used for r in results), total, count, r0.logdet_shift)


def log_likelihood_gsgp_sharded(stats, kg, sigma, opts=None, group=None):
    """log_likelihood_gsgp with the SLQ probes split over the ranks of `group` (every rank holds
    the all-reduced statistics, including every probe image): rank r runs its ⌈P/G⌉ probes,
    the per-probe sums are all-reduced, and every rank returns the same result."""
    import dataclasses

    from .gsgp import LoglikOptions, log_likelihood_gsgp

    opts = opts or LoglikOptions()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    b, e = probe_shard(opts.probes, world, rank)
    if e == b:  # more ranks than probes: an empty shard still takes part in the reduction
        b, e = 0, 0
        mine = dataclasses.replace(opts, probe_begin=0, probe_end=min(1, opts.probes))
        r = log_likelihood_gsgp(stats, kg, sigma, mine)
        r.slq_sum, r.slq_count, r.probes_used = 0.0, 0, 0
    else:
        r = log_likelihood_gsgp(stats, kg, sigma, dataclasses.replace(opts, probe_begin=b, probe_end=e))
    t = torch.tensor([r.slq_sum, float(r.slq_count), float(r.probes_used)], dtype=torch.float64,
                     device=torch.device("cuda", stats.context.device))
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    total, count, used = float(t[0]), int(t[1]), int(t[2])
    r.slq_sum, r.slq_count = total, count
    out = combine_loglik([r], r.quad_term, r.const_term)
    out.probes_used = used
    return out


