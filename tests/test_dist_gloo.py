"""Multi-rank host logic on CPU (world size 2, gloo): the clause-sharded
window protocol of paper_2009_04861_b200.distributed (train_epoch_windows +
torch_allreduce) driven by an oracle-backed shard engine, and sharded class
sums. The GPU engine plugs into the same protocol (GpuShardEngine)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2009_04861_b200 import distributed as D

O_FEAT, M, N, Q = 16, 3, 12, 90


def _data():
    rng = np.random.default_rng(11)
    protos = rng.random((M, O_FEAT)) < 0.4
    y = rng.integers(0, M, Q).astype(np.int32)
    x = (protos[y] ^ (rng.random((Q, O_FEAT)) < 0.1)).astype(np.uint8)
    return x, y


class OracleShardEngine:
    """A rank's clause slice on the CPU oracle: full-size machine/pool
    replicas, but only clauses [jb, je) of every class are trained."""

    def __init__(self, rank, world, seed=3):
        import torch
        self.torch = torch
        x, y = _data()
        self.jb, self.je = D.shard_range(N, rank, world)
        self.tm = O.Machine(O_FEAT, M, N, 8, Q)
        self.pool = O.Pool(x, y, M)
        self.q, self.m, self.seed = Q, M, seed
        self.snap = None

    def begin(self, epoch):
        self.order = O.Rng(self.seed, O.mix_stream(2, epoch)).shuffled_indices(Q)
        self.epoch = epoch

    def window(self, epoch, t0, t1):
        self.snap = self.pool.tallies.copy()
        ev = np.zeros(M, np.uint64)
        for c in range(M):
            for j in range(self.jb, self.je):
                g = c * N + j
                rng = O.Rng(self.seed, O.mix_stream(3, epoch, g) ^ t0)
                off = O.clause_offset(g, Q) + t0
                ev[c] += O.update_clause(self.tm, self.pool, c, j, self.order, off, t1 - t0, 6, 3.0, False, rng)
        return ev

    def delta(self):
        return self.torch.from_numpy((self.pool.tallies - self.snap).reshape(-1).copy())

    def apply(self, reduced):
        own = (self.pool.tallies - self.snap).reshape(-1)
        red = own if reduced is None else reduced.numpy()
        self.pool.tallies[...] = (self.snap.reshape(-1) + red).reshape(Q, M)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = OracleShardEngine(rank, world)
    for e in range(2):
        D.train_epoch_windows(eng, e, windows=5, allreduce=D.torch_allreduce())
    np.save(os.path.join(out_dir, f"tallies{rank}.npy"), eng.pool.tallies)
    np.save(os.path.join(out_dir, f"prev{rank}.npy"), eng.tm.prev)
    np.save(os.path.join(out_dir, f"counters{rank}.npy"), eng.tm.counters)
    # sharded class sums: partial sums over the slice, all-reduced
    import torch
    part = np.zeros((Q, M), np.int64)
    for c in range(M):
        for j in range(eng.jb, eng.je):
            for i in range(Q):
                out = eng.tm.evaluate(c, j, eng.pool.lits[i], 1)
                part[i, c] += out if j % 2 == 0 else -out
    t = torch.from_numpy(part)
    dist.all_reduce(t)
    np.save(os.path.join(out_dir, f"sums{rank}.npy"), t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _bits(prev, q):
    b = np.unpackbits(prev.view(np.uint8), axis=-1, bitorder="little")
    return b[..., :q].astype(np.int64)


def test_window_protocol_two_ranks(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    t0, t1 = np.load(tmp_path / "tallies0.npy"), np.load(tmp_path / "tallies1.npy")
    assert np.array_equal(t0, t1), "replicas diverged after the final all-reduce"
    # global invariant: tally = sum over ALL ranks' clauses of sign(j) * prev bit
    expect = np.zeros((Q, M), np.int64)
    for r in range(world):
        jb, je = D.shard_range(N, r, world)
        bits = _bits(np.load(tmp_path / f"prev{r}.npy"), Q)  # m x n x q
        for c in range(M):
            for j in range(jb, je):
                expect[:, c] += bits[c, j] if j % 2 == 0 else -bits[c, j]
    assert np.array_equal(t0, expect)
    assert np.abs(t0).sum() > 0
    # sharded class sums == class sums of the merged machine
    merged = O.Machine(O_FEAT, M, N, 8)
    counters = np.load(tmp_path / "counters0.npy").copy()
    jb1, je1 = D.shard_range(N, 1, world)
    counters[:, jb1:je1] = np.load(tmp_path / "counters1.npy")[:, jb1:je1]
    merged.set_counters(counters)
    x, _ = _data()
    full = merged.class_sums(O.pack_literals(x))
    assert np.array_equal(np.load(tmp_path / "sums0.npy"), full)
    assert np.array_equal(np.load(tmp_path / "sums1.npy"), full)


def test_single_rank_windows_equal_invariant():
    eng = OracleShardEngine(0, 1)
    D.train_epoch_windows(eng, 0, windows=4, allreduce=None)
    bits = _bits(eng.tm.prev, Q)
    expect = np.stack([(bits[c, 0::2].sum(0) - bits[c, 1::2].sum(0)) for c in range(M)], axis=1)
    assert np.array_equal(eng.pool.tallies, expect)
