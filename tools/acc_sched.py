#!/usr/bin/env python3
"""Asynchronous-schedule experiments on the timed configuration (MNIST-shaped,
q = 60 000, 10 000 test rows, 2000 clauses/class, T = 50, s = 10): 5-seed
mean test accuracy per epoch under the current environment (e.g.
TMG_CLAUSE_ORDER=i), beside the reference's (tests/golden/accuracy_ref.json).
Usage: python tools/acc_sched.py [epochs] [label]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2009_04861_b200 as T  # noqa: E402
from paper_2009_04861_b200 import synth  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
label = sys.argv[2] if len(sys.argv) > 2 else os.environ.get("TMG_CLAUSE_ORDER", "class")
d = synth.make("mnist", 60000, 10000, 2009)
pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
test = T.ExamplePool(784, d.test_x, d.test_y, 10)
acc = np.zeros((5, epochs))
ms = np.zeros((5, epochs))
for k, seed in enumerate(range(1, 6)):
    tm = T.MultiClassTM(T.TMConfig(clauses=2000, margin=50, specificity=10.0, seed=seed), 784, 10)
    pool.reset_tallies()
    for e in range(epochs):
        rep = T.train_epoch_parallel(tm, pool, 8, e)
        ms[k, e] = rep.device_seconds * 1e3
        acc[k, e] = T.evaluate_accuracy(tm, test)
ref = json.load(open(os.path.join(REPO, "tests", "golden", "accuracy_ref.json")))
r = {n: np.mean([ref[n]["per_seed"][s] for s in ref[n]["per_seed"]], axis=0).round(4).tolist()
     for n in ("mnist_q60000", "mnist_q60000_w1", "mnist_q60000_w2", "mnist_q60000_w4") if n in ref}
print(json.dumps({"label": label, "gpu_mean_per_epoch": acc.mean(axis=0).round(4).tolist(),
                  "gpu_std_final": float(acc[:, -1].std().round(4)), "epoch_ms": ms.mean(axis=0).round(2).tolist(),
                  "reference": r}), flush=True)
