#!/usr/bin/env python3
"""Times the W = 1 replay (train_epoch_parallel, workers = 1) with jump-ahead
Type I draws vs serial draws, MNIST-shaped, 200 examples, 200 clauses/class."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2009_04861_b200 as T
from paper_2009_04861_b200 import synth
d = synth.make("mnist", 200, 4, 2009)
res = {}
for mode in ("0", "1"):
    os.environ["TMG_SEQ_SERIAL"] = mode
    tm = T.MultiClassTM(T.TMConfig(clauses=200, margin=50, specificity=10.0, seed=42), 784, 10)
    pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
    t0 = time.perf_counter()
    rep = T.train_epoch_parallel(tm, pool, 1, 0, mode=T.MODE_SYNC_MIRROR)
    res[mode] = time.perf_counter() - t0
    res["dev" + mode] = rep.device_seconds
    res["ev" + mode] = rep.total_feedback_events()
print(json.dumps({"w1_mnist_q200_n200_jump_s": res["0"], "serial_s": res["1"], "speedup": res["1"] / res["0"],
                  "device_s": [res["dev0"], res["dev1"]], "events": [res["ev0"], res["ev1"]]}))
