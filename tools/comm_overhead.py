#!/usr/bin/env python3
"""Overhead of the wave/window exchange on one GPU: the bench's MNIST-shaped
fresh epoch (2000 clauses/class, q = 60 000) as a plain machine, and as a
one-rank NCCL communicator shard (tmg_comm_create with nranks = 1) — the same
code path a rank of the N-GPU bench takes — for several windows per wave.
Usage: python tools/comm_overhead.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_04861_b200 as T  # noqa: E402
from paper_2009_04861_b200 import synth  # noqa: E402

d = synth.make("mnist", 60000, 2000, 2009)
pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
test = T.ExamplePool(784, d.test_x, d.test_y, 10)
cfg = T.TMConfig(clauses=2000, margin=50, specificity=10.0, seed=42)


def run(tm, reps=3):
    out = []
    for r in range(reps + 1):
        tm.reset()
        pool.reset_tallies()
        rep = T.train_epoch_parallel(tm, pool, 8, 0)
        if r:
            out.append(rep.seconds * 1e3)
    return min(out), rep.total_feedback_events(), T.evaluate_accuracy(tm, test)


plain = run(T.MultiClassTM(cfg, 784, 10))
print(json.dumps({"mode": "plain", "ms": plain[0], "events": plain[1], "acc_e0": plain[2]}), flush=True)
comm = T.Comm(T.Comm.unique_id(), 1, 0, 0)
for w in (1, 2, 4, 8, 16):
    tm = T.MultiClassTM(cfg, 784, 10, clause_range=(0, 2000))
    tm.attach_comm(comm)
    tm.set_windows(w)
    r = run(tm)
    print(json.dumps({"mode": "comm1", "windows_per_wave": w, "ms": r[0], "overhead": r[0] / plain[0],
                      "events": r[1], "acc_e0": r[2]}), flush=True)
    tm.attach_comm(None)
