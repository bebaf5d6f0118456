#!/usr/bin/env python3
"""Splits bench.py's e2e step (host buffers through the C ABI) into its phases
on one GPU: pool create (H2D + device packing), reset, epoch, report, destroy."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_04861_b200 as T  # noqa: E402
from paper_2009_04861_b200 import synth  # noqa: E402

d = synth.make("mnist", 60000, 16, 2009)
tm = T.MultiClassTM(T.TMConfig(clauses=2000, margin=50, specificity=10.0, seed=42), 784, 10)
hb = torch.from_numpy(d.train_x).pin_memory().numpy()
hl = torch.from_numpy(d.train_y).pin_memory().numpy()
rows = []
for it in range(4):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    p = T.ExamplePool(784, hb, hl, 10)
    t.append(time.perf_counter())
    tm.reset()
    p.reset_tallies()
    t.append(time.perf_counter())
    rep = T.train_epoch_parallel(tm, p, 1, 0)
    t.append(time.perf_counter())
    _ = [int(v) for v in rep.feedback_events]
    del p
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    rows.append({"pool_ms": (t[1] - t[0]) * 1e3, "reset_ms": (t[2] - t[1]) * 1e3,
                 "epoch_ms": (t[3] - t[2]) * 1e3, "kernel_ms": rep.device_seconds * 1e3,
                 "destroy_ms": (t[4] - t[3]) * 1e3})
print(json.dumps(rows[1:]))
