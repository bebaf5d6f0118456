#!/usr/bin/env python3
"""Phase cycle counts of the grid-wide sequential replay (TMG_STATS build:
TMG_LIB=<variant>/libtmgpu.so). Usage: python tools/seq_phases.py [kind] [q]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2009_04861_b200 as T  # noqa: E402
from paper_2009_04861_b200 import _capi, synth  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "mnist"
q = int(sys.argv[2]) if len(sys.argv) > 2 else 500
T_, s_, seed, n = {"mnist": (50, 10.0, 2009, 2000), "imdb": (100, 15.0, 10000, 10000)}[kind]
d = synth.make(kind, q, 10, seed)
tm = T.MultiClassTM(T.TMConfig(clauses=n, margin=T_, specificity=s_, seed=42), d.features, d.classes)
pool = T.ExamplePool(d.features, d.train_x, d.train_y, d.classes)
c = np.zeros(256, np.uint64)
_capi.check(_capi.lib().tmg_debug_counters(tm.handle, c.ctypes.data, 256, 1))
rep = T.train_epoch_sequential(tm, pool, 0)
_capi.check(_capi.lib().tmg_debug_counters(tm.handle, c.ctypes.data, 256, 1))
names = ["vote+barrier", "scan", "barrier", "apply+barrier", "jumps_in_scan"]
tot = float(sum(int(c[200 + k]) for k in range(4)))
print(json.dumps({"kind": kind, "q": q, "device_s": rep.device_seconds,
                  "us_per_example": {nm: int(c[200 + k]) / 1.965e3 / q for k, nm in enumerate(names)},
                  "share": {nm: int(c[200 + k]) / tot for k, nm in enumerate(names)}}))
