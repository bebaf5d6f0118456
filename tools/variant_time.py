#!/usr/bin/env python3
"""Times the MNIST-shaped fresh async epoch for one libtmgpu.so build.
Usage: TMG_LIB=<path to libtmgpu.so> python tools/variant_time.py [reps] [clauses]
Prints one JSON line: per-epoch device ms (kernel), events, type-I events."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_04861_b200 import _capi  # noqa: E402

import paper_2009_04861_b200 as T  # noqa: E402
from paper_2009_04861_b200 import synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
kind = os.environ.get("TMG_KIND", "mnist")
T_, s_, seed, n0, q0 = {"mnist": (50, 10.0, 2009, 2000, 60000), "fmnist": (100, 15.0, 2352, 8000, 60000),
                        "imdb": (100, 15.0, 10000, 10000, 25000)}[kind]
n = int(sys.argv[2]) if len(sys.argv) > 2 else n0
q = int(sys.argv[3]) if len(sys.argv) > 3 else q0
d = synth.make(kind, q, 2000, seed)
tm = T.MultiClassTM(T.TMConfig(clauses=n, margin=T_, specificity=s_, seed=42), d.features, d.classes)
pool = T.ExamplePool(d.features, d.train_x, d.train_y, d.classes)
test = T.ExamplePool(d.features, d.test_x, d.test_y, d.classes)
ms, ev, ev1 = [], [], []
for r in range(reps + 1):
    tm.reset()
    pool.reset_tallies()
    rep = T.train_epoch_parallel(tm, pool, 1, 0)
    if r:
        ms.append(rep.device_seconds * 1e3)
        ev.append(rep.total_feedback_events())
        ev1.append(sum(rep.type_i_events))
acc0 = T.evaluate_accuracy(tm, test)
rep = T.train_epoch_parallel(tm, pool, 1, 1)
acc1 = T.evaluate_accuracy(tm, test)
print(json.dumps({"lib": _capi.LIB_PATH, "kind": kind, "clauses": n, "q": q, "epoch0_ms": statistics.mean(ms),
                  "epoch0_ms_all": ms, "events": statistics.mean(ev), "type1": statistics.mean(ev1),
                  "epoch1_ms": rep.device_seconds * 1e3, "acc_after_e0": acc0, "acc_after_e1": acc1}))
