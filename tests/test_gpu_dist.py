"""The multi-GPU clause-sharding protocol through torch.distributed with the
REAL GPU engine: two processes (gloo, both on cuda:0 because NCCL refuses
duplicate GPUs and this box has one), GpuShardEngine + torch_allreduce over
CUDA tensors, two epochs; then replicas equal, the tally invariant over both
shards, and sharded class sums equal to the oracle's on the merged machine.
Also runs bench.py's N>1 path the same way (the driver's torchrun launch)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
O_FEAT, M, N, Q = 784, 10, 60, 1500


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, overlapped=False):
    """overlapped: False = synchronous windows, True = overlapped windows,
    "peer" = replicas over peer memory (CUDA IPC; here two processes on one
    GPU)."""
    import torch
    import torch.distributed as dist

    import paper_2009_04861_b200 as T
    from paper_2009_04861_b200 import distributed as D
    from paper_2009_04861_b200 import synth
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    d = synth.make("mnist", Q, 300, 2009)
    jb, je = D.shard_range(N, rank, world)
    tm = T.MultiClassTM(T.TMConfig(clauses=N, margin=20, specificity=10.0, seed=3), O_FEAT, M, clause_range=(jb, je))
    pool = T.ExamplePool(O_FEAT, d.train_x, d.train_y, M)
    eng = D.GpuShardEngine(tm, pool)
    comm = None
    if overlapped == "ipc":  # the engine's own streaming exchange over CUDA IPC (no NCCL)
        def allgather(b):
            out = [None] * world
            dist.all_gather_object(out, b)
            return out
        comm = T.Comm.ipc(world, rank, 0, Q * M, allgather)
        tm.attach_comm(comm)
    if overlapped == "peer":
        assert D.attach_peer_tallies(pool) == world - 1
        try:  # mixing the exchanges would count every tally change twice: refused
            D.train_epoch_overlapped(tm, pool, 0, windows=2)
            raise AssertionError("windowed exchange accepted a pool with peer replicas")
        except ValueError as e:  # std::invalid_argument
            assert "peer tally replicas" in str(e)
    for e in range(2):
        if overlapped == "ipc":
            rep = T.train_epoch_parallel(tm, pool, 8, e)
            assert rep.total_feedback_events() > 0
        elif overlapped == "peer":
            D.train_epoch_peer(tm, pool, e)
        elif overlapped:
            D.train_epoch_overlapped(tm, pool, e, windows=5)
        else:
            D.train_epoch_windows(eng, e, windows=5, allreduce=D.torch_allreduce())
    np.save(os.path.join(out_dir, f"tallies{rank}.npy"), pool.tallies())
    np.save(os.path.join(out_dir, f"prev{rank}.npy"), np.stack([tm.banks[c].prev_outputs() for c in range(M)]))
    np.save(os.path.join(out_dir, f"counters{rank}.npy"), np.stack([tm.banks[c].counters() for c in range(M)]))
    test = T.ExamplePool(O_FEAT, d.test_x, d.test_y, M)
    part = torch.from_numpy(T.class_sums(tm, test).astype(np.int64))
    if comm is None:
        dist.all_reduce(part)
    # (an attached communicator returns the whole machine's sums already)
    np.save(os.path.join(out_dir, f"sums{rank}.npy"), part.numpy())
    if comm is not None:
        tm.attach_comm(None)
        del comm
    dist.barrier()
    dist.destroy_process_group()


def _bits(prev, q):
    b = np.unpackbits(prev.view(np.uint8), axis=-1, bitorder="little")
    return b[..., :q].astype(np.int64)


@pytest.mark.parametrize("overlapped,world", [(False, 2), (True, 2), ("peer", 2), ("peer", 3), ("ipc", 2),
                                              ("ipc", 3)])
def test_gpu_shards_two_processes(tmp_path, overlapped, world):
    """Synchronous windows (train_epoch_windows), the double-buffered,
    overlapped exchange (train_epoch_overlapped) and the peer-memory replicas
    (train_epoch_peer: tally changes added into every replica by the clause
    kernels; also with 3 ranks, two peers per replica) all end each epoch
    with identical replicas satisfying the invariant over all shards."""
    import torch.multiprocessing as mp

    from paper_2009_04861_b200 import distributed as D
    from paper_2009_04861_b200 import synth
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), overlapped), nprocs=world, join=True,
                       start_method="spawn")
    t0 = np.load(tmp_path / "tallies0.npy")
    for r in range(1, world):  # every replica (3 ranks: two peers per replica)
        assert np.array_equal(t0, np.load(tmp_path / f"tallies{r}.npy")), f"replica {r} diverged"
    expect = np.zeros((Q, M), np.int64)
    for r in range(world):
        jb, je = D.shard_range(N, r, world)
        bits = _bits(np.load(tmp_path / f"prev{r}.npy"), Q)  # m x n_loc x q
        for c in range(M):
            for jl in range(je - jb):
                j = jb + jl
                expect[:, c] += bits[c, jl] if j % 2 == 0 else -bits[c, jl]
    assert np.array_equal(t0, expect)
    assert np.abs(t0).sum() > 0
    counters = np.concatenate([np.load(tmp_path / f"counters{r}.npy") for r in range(world)], axis=1)
    merged = O.Machine(O_FEAT, M, N, 128)
    merged.set_counters(counters)
    d = synth.make("mnist", Q, 300, 2009)
    full = merged.class_sums(O.pack_literals(d.test_x))
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"sums{r}.npy"), full)


def _acc_worker(rank, world, port, out_dir, windows):
    import torch
    import torch.distributed as dist

    import paper_2009_04861_b200 as T
    from paper_2009_04861_b200 import distributed as D
    from paper_2009_04861_b200 import synth
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfg = json.load(open(os.path.join(REPO, "tests", "golden", "accuracy_ref.json")))["mnist_q6000"]["config"]
    d = synth.make("mnist", cfg["q"], cfg["qtest"], cfg["data_seed"])
    accs = []
    for seed in range(1, 6):
        jb, je = D.shard_range(cfg["clauses"], rank, world)
        tm = T.MultiClassTM(T.TMConfig(clauses=cfg["clauses"], margin=cfg["T"], specificity=cfg["s"], seed=seed),
                            784, 10, clause_range=(jb, je))
        pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
        if windows == "peer":
            D.attach_peer_tallies(pool)
        for e in range(cfg["epochs"]):
            if windows == "peer":
                D.train_epoch_peer(tm, pool, e)
            else:
                D.train_epoch_overlapped(tm, pool, e, windows=windows)
        if windows == "peer":
            D.detach_peer_tallies(pool)
            dist.barrier()
        test = T.ExamplePool(784, d.test_x, d.test_y, 10)
        part = torch.from_numpy(T.class_sums(tm, test).astype(np.int64))
        dist.all_reduce(part)
        accs.append(float((part.numpy().argmax(1) == d.test_y).mean()))
    if rank == 0:
        json.dump(accs, open(os.path.join(out_dir, "accs.json"), "w"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", [16, "peer"])
def test_two_rank_accuracy_parity(tmp_path, exchange):
    """Clause-sharded training (2 ranks x 1000 clauses/class, MNIST-shaped
    q = 6000, 3 epochs, 5 seeds; overlapped 16-window exchange, or the
    peer-memory replicas) matches the reference's multi-threaded trainer on
    the same data within 0.5 pt — the multi-GPU staleness does not cost
    accuracy."""
    import torch.multiprocessing as mp
    ref = json.load(open(os.path.join(REPO, "tests", "golden", "accuracy_ref.json")))["mnist_q6000"]
    mp.start_processes(_acc_worker, args=(2, _free_port(), str(tmp_path), exchange), nprocs=2, join=True,
                       start_method="spawn")
    accs = json.load(open(tmp_path / "accs.json"))
    from tests.test_gpu_async import accuracy_parity
    ok, msg = accuracy_parity("mnist_q6000", accs)
    print("2-rank sharded " + msg)
    assert ok, msg


@pytest.mark.parametrize("exchange,expect", [("ipc", "ipc"), ("comm", "ipc"), ("peer", "peer")])
def test_bench_two_ranks_protocol(exchange, expect):
    """bench.py under torchrun with 2 ranks (gloo, shared device): one JSON
    line from rank 0 with n_gpus = 2 and a positive value. The default
    exchange (the engine's communicator over CUDA IPC) runs as it would on
    two GPUs; the NCCL one needs one GPU per rank, so on a shared device it
    falls back to IPC and says so."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(REPO, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "1", "--no-cpu", "--dist-backend", "gloo", "--share-device",
           "--exchange", exchange]
    out = subprocess.run(cmd, check=True, capture_output=True, text=True, timeout=900, cwd=REPO).stdout
    lines = [json.loads(l) for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == 2 and lines[0]["value"] > 0
    assert lines[0]["config"]["clauses_per_class_total"] == 4000
    assert lines[0]["config"]["exchange"] == expect
    if exchange == "comm":
        assert "NCCL" in lines[0]["config"]["exchange_note"]
    if expect == "ipc":  # the engine's exchange reported every rank's events
        assert lines[0]["feedback_events_per_step"] > 0
