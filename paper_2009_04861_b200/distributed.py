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

The fused alternative (attach_peer_tallies / train_epoch_peer): every rank's
replica is mapped into every other rank over CUDA IPC, and the training
kernels add each tally change into all replicas as it happens (NVLink
reductions inside the clause kernel) — no windows, no collective call, and a
staleness of one NVLink round trip instead of one window.

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


class GpuShardEngine:
    """One rank's clause shard on its GPU (the product engine)."""

    def __init__(self, tm: MultiClassTM, pool: ExamplePool):
        self.tm, self.pool = tm, pool
        self.q, self.m = pool.size(), tm.num_banks()

    def begin(self, epoch: int):
        check(lib().tmg_epoch_begin(self.tm.handle, self.pool.handle, epoch))

    def window(self, epoch: int, t0: int, t1: int) -> np.ndarray:
        ev = np.zeros(self.m, np.uint64)
        check(lib().tmg_train_window(self.tm.handle, self.pool.handle, epoch, t0, t1, ev.ctypes.data))
        return ev

    def delta(self):
        return torch_view(self.pool.delta_device_ptr(), self.q * self.m, self.pool.device)

    def apply(self, reduced):
        ptr = reduced.data_ptr() if reduced is not None else self.pool.delta_device_ptr()
        check(lib().tmg_pool_apply_reduced(self.pool.handle, C.c_void_p(ptr)))


def torch_allreduce(group=None) -> Callable:
    """Sum of the per-rank delta buffers (NCCL for CUDA tensors, gloo for CPU)."""
    import torch
    import torch.distributed as dist

    def run(own):
        red = own.clone()
        dist.all_reduce(red, op=dist.ReduceOp.SUM, group=group)
        if red.is_cuda:
            torch.cuda.synchronize(red.device)
        return red

    return run


def train_epoch_windows(engine, epoch: int, windows: int, allreduce: Optional[Callable]) -> List[int]:
    """One asynchronous epoch as `windows` windows of every clause's pass.

    After each window: reduced = allreduce(own delta); replica += reduced - own;
    own = 0. With allreduce=None (one rank) the remote share is zero."""
    engine.begin(epoch)
    total = np.zeros(engine.m, np.uint64)
    for t0, t1 in window_bounds(engine.q, windows):
        total += engine.window(epoch, t0, t1)
        reduced = allreduce(engine.delta()) if allreduce is not None else None
        engine.apply(reduced)
    return [int(v) for v in total]


def train_epoch_overlapped(tm: MultiClassTM, pool: ExamplePool, epoch: int, windows: int, group=None,
                           comm_stream=None) -> List[int]:
    """One asynchronous epoch as `windows` windows with the tally exchange
    double-buffered and overlapped: the window kernels run
    back to back on the machine's stream; after window w its own deltas are
    snapshotted (and zeroed) on that stream, all-reduced on a side stream
    while window w+1 runs, and the remote share (reduced - own) of window w is
    added before window w+2 — one window more staleness than
    train_epoch_windows and no host round trip per window. With one rank
    (group world size 1 / no process group) the exchange is skipped."""
    import torch
    import torch.distributed as dist

    from .tsetlin import machine_stream
    device = pool.device
    q, m = pool.size(), tm.num_banks()
    multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
    ms = torch.cuda.ExternalStream(machine_stream(tm), device=f"cuda:{device}")
    cs = comm_stream if comm_stream is not None else torch.cuda.Stream(device=f"cuda:{device}")
    snaps = [torch.empty(q * m, dtype=torch.int32, device=f"cuda:{device}") for _ in range(2)]
    reds = [torch.empty_like(snaps[0]) for _ in range(2)]
    done = [None, None]
    check(lib().tmg_epoch_begin(tm.handle, pool.handle, epoch))
    bounds = window_bounds(q, windows)
    for w, (t0, t1) in enumerate(bounds):
        b = w % 2
        check(lib().tmg_train_window_async(tm.handle, pool.handle, epoch, t0, t1))
        check(lib().tmg_window_delta_snapshot(tm.handle, pool.handle, C.c_void_p(snaps[b].data_ptr())))
        if multi:
            ready = torch.cuda.Event()
            ready.record(ms)
            with torch.cuda.stream(cs):
                cs.wait_event(ready)
                reds[b].copy_(snaps[b])
                dist.all_reduce(reds[b], op=dist.ReduceOp.SUM, group=group)
                done[b] = torch.cuda.Event()
                done[b].record(cs)
            if w >= 1:
                p = (w - 1) % 2
                ms.wait_event(done[p])
                check(lib().tmg_window_apply_remote(tm.handle, pool.handle, C.c_void_p(reds[p].data_ptr()),
                                                    C.c_void_p(snaps[p].data_ptr())))
    if multi and bounds:
        p = (len(bounds) - 1) % 2
        ms.wait_event(done[p])
        check(lib().tmg_window_apply_remote(tm.handle, pool.handle, C.c_void_p(reds[p].data_ptr()),
                                            C.c_void_p(snaps[p].data_ptr())))
    ev = np.zeros(m, np.uint64)
    check(lib().tmg_epoch_events(tm.handle, ev.ctypes.data))
    return [int(v) for v in ev]


def attach_peer_tallies(pool: ExamplePool, group=None) -> int:
    """Peer-memory exchange, the fused alternative to the
    windowed all-reduce: every rank exports its pool's tally replica
    (cudaIpcMemHandle, gathered over the process group) and opens the others',
    after which the training kernels add every tally change into all replicas
    over NVLink as it happens. Returns the number of peers attached. Raises
    TMError when a handle cannot be opened (no P2P path between the GPUs);
    callers fall back to train_epoch_overlapped."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world - 1 > 7:
        raise ValueError("peer-memory exchange supports up to 8 ranks (one node)")
    h = (C.c_ubyte * 64)()
    check(lib().tmg_pool_tally_ipc_handle(pool.handle, h))
    handles = [None] * world
    dist.all_gather_object(handles, bytes(h), group=group)
    others = b"".join(handles[r] for r in range(world) if r != rank)
    buf = (C.c_ubyte * max(1, len(others))).from_buffer_copy(others or b"\0")
    check(lib().tmg_pool_set_peers(pool.handle, buf, world - 1))
    return world - 1


def detach_peer_tallies(pool: ExamplePool) -> None:
    check(lib().tmg_pool_set_peers(pool.handle, None, 0))


def train_epoch_peer(tm: MultiClassTM, pool: ExamplePool, epoch: int, group=None) -> List[int]:
    """One asynchronous epoch of this rank's clause shard with the tally
    replicas attached by attach_peer_tallies: a barrier so that no rank adds
    into a replica that another rank is still resetting, the epoch (the
    kernels keep every replica current), and a barrier so that every rank's
    remote adds have landed before anyone reads its tallies. Every replica
    then holds the same tallies, over all shards."""
    import torch
    import torch.distributed as dist
    from .tsetlin import MODE_ASYNC, train_epoch_parallel
    torch.cuda.synchronize(pool.device)
    dist.barrier(group=group)
    rep = train_epoch_parallel(tm, pool, 1, epoch, mode=MODE_ASYNC)
    torch.cuda.synchronize(pool.device)
    dist.barrier(group=group)
    return [int(v) for v in rep.feedback_events]


def nccl_allreduce(device: int, group=None) -> Callable:
    return torch_allreduce(group)


def class_sums_sharded(tm: MultiClassTM, pool: ExamplePool, mode: int, allreduce_host: Callable):
    """Per-shard partial class sums, summed across ranks (bit-exact: integers)."""
    part = class_sums(tm, pool, mode)
    return allreduce_host(part)
