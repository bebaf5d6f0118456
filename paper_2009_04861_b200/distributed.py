"""Clause sharding across GPUs (one process per GPU, torch.distributed/NCCL).

Every rank owns an even-aligned slice of every class's clauses
(SURVEY.md §8(e)); the example pool, labels and the q x m tally array are
replicated. An epoch is cut into windows of each clause's pass: a window runs
the asynchronous kernel locally (tally deltas go to the local replica AND to
a delta buffer), then the delta buffers are summed with one all-reduce and the
remote share (reduced - own) is added to each replica. Between windows a rank
sees other ranks' clause outputs with at most one window of extra staleness —
the same relaxed, lock-free tally semantics as the reference's worker threads
(pool.hpp:54-62), now across NVLink.

Clause keys (RNG counters, per-clause offsets) use the GLOBAL clause index, so
sampling does not depend on the number of ranks.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, List, Optional, Tuple

import numpy as np

from ._capi import check, lib
from .tsetlin import ExamplePool, MultiClassTM, class_sums


def shard_range(clauses: int, rank: int, world: int) -> Tuple[int, int]:
    """Even-aligned contiguous slice [jb, je) of `clauses` for `rank`.

    Pairs (2k, 2k+1) are never split so each shard keeps the alternating
    +/- polarity balance (core.hpp:122-124)."""
    if clauses % 2:
        raise ValueError("clauses must be even")
    pairs = clauses // 2
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if pairs < world:
        raise ValueError("fewer clause pairs than ranks")
    base, extra = divmod(pairs, world)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return 2 * start, 2 * (start + count)


def window_bounds(q: int, windows: int) -> List[Tuple[int, int]]:
    windows = max(1, min(windows, q))
    edges = [q * k // windows for k in range(windows + 1)]
    return [(edges[k], edges[k + 1]) for k in range(windows)]


class _CudaArray:
    """Zero-copy __cuda_array_interface__ view of a device int32 buffer."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<i4", "data": (ptr, False),
                                         "version": 3, "strides": None}


def torch_view(ptr: int, count: int, device: int):
    import torch
    return torch.as_tensor(_CudaArray(ptr, count), device=f"cuda:{device}")


def nccl_allreduce(device: int, group=None) -> Callable:
    """All-reduce of the pool's tally-delta buffer with torch.distributed."""
    import torch
    import torch.distributed as dist

    def run(delta_ptr: int, count: int):
        own = torch_view(delta_ptr, count, device)
        red = own.clone()
        dist.all_reduce(red, op=dist.ReduceOp.SUM, group=group)
        torch.cuda.synchronize(device)
        return red

    return run


def train_epoch_windows(tm: MultiClassTM, pool: ExamplePool, epoch: int, windows: int,
                        allreduce: Optional[Callable]) -> List[int]:
    """One asynchronous epoch as `windows` windows; `allreduce(delta_ptr,
    count)` returns the summed delta (a tensor) or None for a single rank."""
    check(lib().tmg_epoch_begin(tm.handle, pool.handle, epoch))
    m, q = tm.num_banks(), pool.size()
    total = np.zeros(m, np.uint64)
    ev = np.zeros(m, np.uint64)
    delta_ptr = pool.delta_device_ptr()
    for t0, t1 in window_bounds(q, windows):
        check(lib().tmg_train_window(tm.handle, pool.handle, epoch, t0, t1, ev.ctypes.data))
        total += ev
        reduced = allreduce(delta_ptr, q * m) if allreduce is not None else None
        if reduced is None:
            check(lib().tmg_pool_apply_reduced(pool.handle, C.c_void_p(delta_ptr)))  # remote = 0
        else:
            check(lib().tmg_pool_apply_reduced(pool.handle, C.c_void_p(reduced.data_ptr())))
    return [int(v) for v in total]


def class_sums_sharded(tm: MultiClassTM, pool: ExamplePool, mode: int, allreduce_host: Callable):
    """Per-shard partial class sums, summed across ranks (bit-exact: integers)."""
    part = class_sums(tm, pool, mode)
    return allreduce_host(part)
