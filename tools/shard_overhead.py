#!/usr/bin/env python3
"""Cost of the clause-sharded machinery (csrc/group.cu) on ONE GPU: a machine
of S x 2000 clauses/class held as S shards on cuda:0 (windowed exchange,
peer-memory sums, one tally replica per shard) against the same clause count
as one plain machine, MNIST-shaped fresh epoch, q = 60 000. The ratio is the
protocol's own overhead (window tails, snapshot/sum/apply kernels, replica
syncs); it is not multi-GPU scaling — the shards share one GPU's SMs.
Usage: python tools/shard_overhead.py [shards ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_04861_b200 as T  # noqa: E402
from paper_2009_04861_b200 import synth  # noqa: E402

d = synth.make("mnist", 60000, 2000, 2009)
pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
test = T.ExamplePool(784, d.test_x, d.test_y, 10)


def epoch_s(tm, reps=3):
    out = []
    for r in range(reps + 1):
        tm.reset()
        pool.reset_tallies()
        t0 = time.perf_counter()
        rep = T.train_epoch_parallel(tm, pool, 8, 0)
        if r:
            out.append(time.perf_counter() - t0)
    return min(out), rep.total_feedback_events(), T.evaluate_accuracy(tm, test)


for s in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]:
    cfg = T.TMConfig(clauses=2000 * s, margin=50, specificity=10.0, seed=42)
    plain = epoch_s(T.MultiClassTM(cfg, 784, 10))
    sharded = epoch_s(T.MultiClassTM(cfg, 784, 10, devices=[0] * s)) if s > 1 else plain
    print(json.dumps({"shards_on_one_gpu": s, "clauses_per_class": 2000 * s, "plain_ms": plain[0] * 1e3,
                      "sharded_ms": sharded[0] * 1e3, "overhead": sharded[0] / plain[0],
                      "plain_events": plain[1], "sharded_events": sharded[1],
                      "plain_acc_e0": plain[2], "sharded_acc_e0": sharded[2]}), flush=True)
