#!/usr/bin/env python3
"""Inference (class sums / predict_all, trainer.cpp:262-279, pool.cpp:82-91)
on machines trained for one async epoch at the MNIST / FMNIST / IMDb shapes
of BASELINE.json configs[1..3]: device time of the class-sum kernels on the
full test split (CUDA events on the engine stream, literal lists rebuilt and
example columns transposed inside the timed call), and a numpy check of the
class sums on a row sample computed from the machine's own counters.

Usage: python tools/eval_bench.py [mnist fmnist imdb] > gpurun_out/eval.jsonl
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_04861_b200 as T  # noqa: E402
from paper_2009_04861_b200 import _capi, synth  # noqa: E402
from paper_2009_04861_b200.tsetlin import machine_stream  # noqa: E402

SHAPES = {
    "mnist": dict(o=784, m=10, n=2000, T=50, s=10.0, q=60000, qt=10000, seed=2009),
    "fmnist": dict(o=2352, m=10, n=8000, T=100, s=15.0, q=60000, qt=10000, seed=2352),
    "imdb": dict(o=10000, m=2, n=10000, T=100, s=15.0, q=25000, qt=25000, seed=10000),
}


def numpy_sums(counters, lits_bits, N, o):
    """vote_sum (pool.cpp:82-91) for every class: counters [m][n][2o], rows [r][o] 0/1."""
    r = lits_bits.shape[0]
    lit = np.concatenate([lits_bits, 1 - lits_bits], axis=1).astype(np.float32)  # [r][2o]
    out = np.zeros((r, counters.shape[0]), np.int64)
    for c in range(counters.shape[0]):
        inc = (counters[c] > N).astype(np.float32)  # [n][2o]
        viol = inc @ (1.0 - lit).T  # [n][r] count of falsified included literals
        nonempty = inc.sum(axis=1) > 0
        fire = (viol == 0) & nonempty[:, None]
        sign = np.where(np.arange(inc.shape[0]) % 2 == 0, 1, -1)
        out[:, c] = (fire * sign[:, None]).sum(axis=0)
    return out


def run(name, epochs=1, check_rows=256):
    p = SHAPES[name]
    d = synth.make(name, p["q"], p["qt"], p["seed"])
    tm = T.MultiClassTM(T.TMConfig(clauses=p["n"], margin=p["T"], specificity=p["s"], seed=42), p["o"], p["m"])
    pool = T.ExamplePool(p["o"], d.train_x, d.train_y, p["m"])
    t0 = time.time()
    for e in range(epochs):
        T.train_epoch_parallel(tm, pool, 1, e)
    train_s = time.time() - t0
    del pool
    test = T.ExamplePool(p["o"], d.test_x, d.test_y, p["m"])
    qt = p["qt"]
    sums = torch.zeros(qt * p["m"], dtype=torch.int32, device="cuda:0")
    stream = torch.cuda.ExternalStream(machine_stream(tm), device="cuda:0")
    ms = []
    for r in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _capi.check(_capi.lib().tmg_class_sums_device(tm.handle, test.handle, T.PREDICT, sums.data_ptr()))
        e1.record(stream)
        torch.cuda.synchronize()
        if r:
            ms.append(e0.elapsed_time(e1))
    t0 = time.perf_counter()
    pred = T.predict_all(tm, test)
    predict_call_ms = (time.perf_counter() - t0) * 1e3
    gpu = sums.view(qt, p["m"]).cpu().numpy()
    counters = np.stack([b.counters() for b in tm.banks])
    inc = (counters > tm.config.state_depth).sum(axis=2)
    ref = numpy_sums(counters, d.test_x[:check_rows].astype(np.int64), tm.config.state_depth, p["o"])
    argmax_ok = bool(np.array_equal(pred, np.argmax(gpu, axis=1) if p["m"] > 1 else (gpu[:, 0] >= 0)))
    dense_lop3 = p["m"] * p["n"] * qt * ((2 * p["o"] + 31) // 32)
    out = dict(shape=name, clauses_per_class=p["n"], test_rows=qt, epochs_trained=epochs, train_s=train_s,
               class_sums_ms_min=min(ms), class_sums_ms_median=float(np.median(ms)),
               predict_call_ms=predict_call_ms, rows_per_s=qt / (min(ms) * 1e-3),
               dense_lop3_equiv_per_s=dense_lop3 / (min(ms) * 1e-3),
               mean_included_literals=float(inc.mean()), max_included_literals=int(inc.max()),
               accuracy=float((pred == d.test_y).mean()),
               sums_match_numpy=bool(np.array_equal(gpu[:check_rows], ref)), argmax_consistent=argmax_ok)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or list(SHAPES):
        run(nm)
