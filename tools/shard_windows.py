#!/usr/bin/env python3
"""Sharded-machine staleness: epoch-0..2 test accuracy of 2000 clauses/class
held as S shards on cuda:0 with W exchange windows per epoch, vs one machine
(MNIST-shaped, q = 60 000). Usage: python tools/shard_windows.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_04861_b200 as T  # noqa: E402
from paper_2009_04861_b200 import synth  # noqa: E402

d = synth.make("mnist", 60000, 2000, 2009)
pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
test = T.ExamplePool(784, d.test_x, d.test_y, 10)
for shards, windows in [(1, 1), (2, 4), (2, 16), (2, 64), (2, 256), (4, 16), (4, 256)]:
    cfg = T.TMConfig(clauses=2000, margin=50, specificity=10.0, seed=42)
    tm = T.MultiClassTM(cfg, 784, 10, devices=[0] * shards) if shards > 1 else T.MultiClassTM(cfg, 784, 10)
    if shards > 1:
        tm.set_windows(windows)
    pool.reset_tallies()
    acc, ev, ms = [], [], []
    for e in range(3):
        rep = T.train_epoch_parallel(tm, pool, 8, e)
        acc.append(round(T.evaluate_accuracy(tm, test), 4))
        ev.append(rep.total_feedback_events())
        ms.append(round(rep.seconds * 1e3, 1))
    print(json.dumps({"shards": shards, "windows": windows, "acc": acc, "events": ev, "ms": ms}), flush=True)
