#!/usr/bin/env python3
"""Type I draw statistics of a fresh MNIST-shaped async epoch, from a
TMG_STATS build (TMG_LIB=<variant>/libtmgpu.so): per clause output, how many
of a warp's literal draws can move an automaton (not already saturated in the
direction of the step), as the warp maximum per lane and the warp total."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_04861_b200 import _capi  # noqa: E402

import paper_2009_04861_b200 as T  # noqa: E402
from paper_2009_04861_b200 import synth  # noqa: E402

d = synth.make("mnist", 60000, 16, 2009)
tm = T.MultiClassTM(T.TMConfig(clauses=2000, margin=50, specificity=10.0, seed=42), 784, 10)
pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
out = {}
for e in range(3):
    T.train_epoch_parallel(tm, pool, 1, e)
    c = np.zeros(256, np.uint64)
    _capi.check(_capi.lib().tmg_debug_counters(tm.handle, c.ctypes.data, 256, 1))
    for name, base in (("out0", 0), ("out1", 128)):
        ev = int(c[base + 64])
        hist = c[base:base + 64].astype(np.float64)
        cdf = np.cumsum(hist) / max(ev, 1)
        out[f"e{e}_{name}"] = {"events": ev, "relevant_per_warp": float(c[base + 65]) / max(ev, 1),
                               "mean_lane_max": float(c[base + 66]) / max(ev, 1),
                               "p_lane_max_le": {k: round(float(cdf[k]), 4) for k in (2, 4, 8, 12, 16, 24, 32)}}
print(json.dumps(out, indent=1))
