"""Clause-sharded machines through the C ABI
(paper_2009_04861_b200/csrc/group.cu): one process driving several shards
(tmg_machine_create_devices; on this one-GPU box the shards share cuda:0 and
sum their tally deltas with the peer-memory reduction kernel), and one rank's
shard on an NCCL communicator (tmg_comm_create, exercised with one rank).

Reference: train_epoch_parallel's workers share one tally array through
relaxed atomics (trainer.cpp:210-231, pool.hpp:57-59); here every shard keeps
a replica and the replicas exchange deltas every window."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

T = pytest.importorskip("paper_2009_04861_b200")
from paper_2009_04861_b200 import synth  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(REPO, "paper_2009_04861_b200", "_lib")


def _invariant(tm, pool, n):
    """tally[i][c] == sum_j sign(j) prev[c][j][i] (record_output_and_tally, pool.cpp:93-106)."""
    q = pool.size()
    tal = pool.tallies()
    for c in range(tm.num_banks()):
        prev = tm.banks[c].prev_outputs()
        bits = np.unpackbits(prev.view(np.uint8), axis=1, bitorder="little")[:, :q].astype(np.int64)
        sign = np.where(np.arange(n) % 2 == 0, 1, -1)
        assert np.array_equal((bits * sign[:, None]).sum(axis=0), tal[:, c]), f"bank {c}"


@pytest.mark.parametrize("devices", ["0,0", "0,0,0"])
def test_shard_driver_through_c_abi(devices):
    """tests/cpp/shard_driver.cpp (C ABI only): replicas equal and the tally
    invariant after every epoch, sharded class sums == one-device sums."""
    out = subprocess.run([os.path.join(LIB, "shard_driver"), devices, "1000", "3"], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().endswith("OK")
    acc = float(out.stdout.split("accuracy")[1].split()[0])
    assert acc > 0.7, out.stdout  # 1000 clauses/class, q = 6000, 3 epochs (unsharded: ~0.85)


def test_sharded_machine_python_api():
    d = synth.make("mnist", 6000, 2000, 2009)
    cfg = T.TMConfig(clauses=400, margin=50, specificity=10.0, seed=42)
    tm = T.MultiClassTM(cfg, 784, 10, devices=[0, 0])
    assert tm.exchange_info() == (2, False)
    pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
    test = T.ExamplePool(784, d.test_x, d.test_y, 10)
    for e in range(3):
        rep = T.train_epoch_parallel(tm, pool, 8, e)
        assert rep.total_feedback_events() > 0 and sum(rep.type_i_events) > 0
        _invariant(tm, pool, 400)
    acc = T.evaluate_accuracy(tm, test)
    # the same automata on one device: identical sums / predictions / refresh
    one = T.MultiClassTM(cfg, 784, 10)
    for c in range(10):
        one.banks[c].set_counters(tm.banks[c].counters())
        assert np.array_equal(tm.banks[c].include_counts(), one.banks[c].include_counts())
        assert np.array_equal(tm.banks[c].include_masks(), one.banks[c].include_masks())
    assert np.array_equal(T.class_sums(tm, test), T.class_sums(one, test))
    assert np.array_equal(T.predict_all(tm, test), T.predict_all(one, test))
    lits = test.all_literals()[:7]
    assert np.array_equal(T.export_vote_sums(tm, lits), T.export_vote_sums(one, lits))
    pool2 = T.ExamplePool(784, d.train_x, d.train_y, 10)
    T.refresh_tallies(pool, tm)
    T.refresh_tallies(pool2, one)
    assert np.array_equal(pool.tallies(), pool2.tallies())
    for c in range(10):
        assert np.array_equal(tm.banks[c].prev_outputs(), one.banks[c].prev_outputs())
    # per-clause calls go to the shard that owns the clause
    for j in (0, 1, 250, 399):
        assert T.evaluate_clause(tm.banks[3], j, lits[0], T.TRAIN) == T.evaluate_clause(one.banks[3], j, lits[0],
                                                                                         T.TRAIN)
    # calls that replay the reference's serial streams need one device
    with pytest.raises(ValueError, match="single-device"):
        T.train_epoch_sequential(tm, pool, 0)
    with pytest.raises(ValueError, match="asynchronously"):
        T.train_epoch_parallel(tm, pool, 1, 0, mode=T.MODE_SYNC_MIRROR)
    assert acc > 0.45  # 400 clauses/class learn slowly (unsharded: 0.53 after 3 epochs, tools/shard_acc.py)


def test_sharded_accuracy_matches_unsharded():
    """Two shards exchanging every 16th of a pass learn like one machine
    (MNIST-shaped, 2000 clauses/class, q = 6000, 3 epochs, mean of 3 seeds)."""
    d = synth.make("mnist", 6000, 2000, 2009)
    accs = {1: [], 2: []}
    for seed in (1, 2, 3):
        for shards in (1, 2):
            cfg = T.TMConfig(clauses=2000, margin=50, specificity=10.0, seed=seed)
            tm = T.MultiClassTM(cfg, 784, 10, devices=[0] * shards)
            pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
            for e in range(3):
                T.train_epoch_parallel(tm, pool, 8, e)
            accs[shards].append(T.evaluate_accuracy(tm, T.ExamplePool(784, d.test_x, d.test_y, 10)))
    m1, m2 = np.mean(accs[1]), np.mean(accs[2])
    assert abs(m1 - m2) <= 0.01, accs


def test_one_rank_nccl_communicator():
    """The multi-process path (tmg_comm_create + attach) with one rank: NCCL
    init, the windowed all-reduce and the event all-reduce run for real."""
    ok, why = T.nccl_available()
    if not ok:
        pytest.skip(why)
    d = synth.make("mnist", 3000, 1000, 2009)
    cfg = T.TMConfig(clauses=200, margin=50, specificity=10.0, seed=5)
    tm = T.MultiClassTM(cfg, 784, 10, clause_range=(0, 200))
    comm = T.Comm(T.Comm.unique_id(), 1, 0, 0)
    tm.attach_comm(comm)
    assert tm.exchange_info() == (1, True)
    pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
    for e in range(2):
        rep = T.train_epoch_parallel(tm, pool, 8, e)
        assert rep.total_feedback_events() > 0
        _invariant(tm, pool, 200)
    test = T.ExamplePool(784, d.test_x, d.test_y, 10)
    sums = T.class_sums(tm, test)
    tm.attach_comm(None)
    assert np.array_equal(sums, T.class_sums(tm, test))
    del comm


def test_facade_spans_devices(tmp_path):
    """The C++ facade with TSETLIN_DEVICES=0,0: MultiClassTM is a two-shard
    machine behind the reference's API (`tm train --mode par`)."""
    env = {k: v for k, v in os.environ.items() if k not in ("TM_THREADS", "TSETLIN_DETERMINISTIC")}
    env["TSETLIN_DEVICES"] = "0,0"
    p = subprocess.run([os.path.join(LIB, "tm"), "train", "--synth", "patterns", "--synth-train", "2000",
                        "--synth-test", "500", "--classes", "4", "--clauses", "40", "--epochs", "5", "--mode", "par",
                        "--workers", "8", "--out", str(tmp_path / "m.model")],
                       capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, p.stderr
    vals = dict(l.split(" ", 1) for l in p.stdout.splitlines() if " " in l)
    assert float(vals["test_accuracy"]) >= 0.9, p.stdout
    e = subprocess.run([os.path.join(LIB, "tm"), "train", "--synth", "patterns", "--synth-train", "200",
                        "--synth-test", "50", "--classes", "4", "--clauses", "40", "--epochs", "1", "--mode", "seq"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert e.returncode == 1 and "single-device" in e.stderr
