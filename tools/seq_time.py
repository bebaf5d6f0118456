#!/usr/bin/env python3
"""Times train_epoch_sequential (the bit-exact GPU replay of the reference's
classic trainer) on a q-prefix of a config's synthetic data,
parallel replay vs serial replay (TMG_SEQ_SERIAL=1), and checks that both
leave identical automaton states. Usage: python tools/seq_time.py [kind] [q] [clauses]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2009_04861_b200 as T  # noqa: E402
from paper_2009_04861_b200 import synth  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "mnist"
q = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
T_, s_, seed, n0 = {"mnist": (50, 10.0, 2009, 2000), "fmnist": (100, 15.0, 2352, 8000),
                    "imdb": (100, 15.0, 10000, 10000), "xor": (15, 3.9, 1, 20)}[kind]
n = int(sys.argv[3]) if len(sys.argv) > 3 else n0
d = synth.make(kind, q, 10, seed)
out = {"kind": kind, "q": q, "clauses": n}
states = {}
for mode in ("parallel", "serial"):
    os.environ["TMG_SEQ_SERIAL"] = "1" if mode == "serial" else "0"
    tm = T.MultiClassTM(T.TMConfig(clauses=n, margin=T_, specificity=s_, seed=42), d.features, d.classes)
    pool = T.ExamplePool(d.features, d.train_x, d.train_y, d.classes)
    t0 = time.perf_counter()
    rep = T.train_epoch_sequential(tm, pool, 0)
    out[f"{mode}_s"] = time.perf_counter() - t0
    out[f"{mode}_events"] = rep.total_feedback_events()
    states[mode] = np.stack([tm.banks[c].counters() for c in range(d.classes)])
out["identical"] = bool(np.array_equal(states["parallel"], states["serial"]))
out["speedup"] = out["serial_s"] / out["parallel_s"]
print(json.dumps(out))
