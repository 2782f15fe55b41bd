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
    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


def stats_buffer_tensor(stats, device=None) -> torch.Tensor:
    """A torch view (no copy) of the stats' reduce buffer."""
    ptr, count = stats.reduce_buffer()
    dev = device if device is not None else torch.device("cuda", stats.context.device)
    return torch.as_tensor(_DevView(ptr, count), device=dev)


def allreduce_stats(stats, group=None):
    """Sum the finalized statistics of every rank in place (all ranks end with the merged
    statistics) and mark the object reduced."""
    buf = stats_buffer_tensor(stats)
    stats.context.synchronize()
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    torch.cuda.current_stream(buf.device).synchronize()
    stats.mark_reduced()
    return stats


def merge_buffers_host(buffers):
    """Host restatement of the combine step (used by the gloo CPU tests)."""
    out = buffers[0].clone()
    for b in buffers[1:]:
        out += b
    return out
