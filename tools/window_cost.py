#!/usr/bin/env python3
"""Cost of cutting an async epoch into tally-exchange windows (the multi-GPU
protocol, distributed.py) on ONE GPU: epoch time for 1..64 windows with no
remote ranks, host-synchronous (train_epoch_windows) and double-buffered
(train_epoch_overlapped), MNIST shape, fresh machine each time (wall clock,
synchronised)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_04861_b200 as T  # noqa: E402
from paper_2009_04861_b200 import distributed as D  # noqa: E402
from paper_2009_04861_b200 import synth  # noqa: E402

d = synth.make("mnist", 60000, 16, 2009)
tm = T.MultiClassTM(T.TMConfig(clauses=2000, margin=50, specificity=10.0, seed=42), 784, 10)
pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
eng = D.GpuShardEngine(tm, pool)
out = {}
for mode in ("sync", "overlapped"):
    for w in [1, 4, 16, 64]:
        ts = []
        for r in range(3):
            tm.reset()
            pool.reset_tallies()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if mode == "sync":
                ev = D.train_epoch_windows(eng, 0, w, None)
            else:
                ev = D.train_epoch_overlapped(tm, pool, 0, w)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        out[f"{mode}_{w}"] = {"ms": min(ts[1:]), "events": sum(ev)}
print(json.dumps(out))
