#!/usr/bin/env python3
"""Inference throughput (class sums / predict_all) on a trained MNIST-shaped
machine: the GPU's eval kernel on the 10 000 test rows (device time, CUDA
events on the engine stream) vs the reference's single-threaded predict_all on
the SAME model file (tmmodel v1) for a bounded row sample, with the
predictions compared row for row."""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2009_04861_b200 import _capi  # noqa: E402

import paper_2009_04861_b200 as T  # noqa: E402
from paper_2009_04861_b200 import model_io, synth  # noqa: E402
from paper_2009_04861_b200.tsetlin import machine_stream  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ref_rows = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
q, qt, seed = 60000, 10000, 2009
d = synth.make("mnist", q, qt, seed)
tm = T.MultiClassTM(T.TMConfig(clauses=n, margin=50, specificity=10.0, seed=42), 784, 10)
pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
for e in range(epochs):
    T.train_epoch_parallel(tm, pool, 1, e)
test = T.ExamplePool(784, d.test_x, d.test_y, 10)
sums = torch.zeros(qt * 10, dtype=torch.int32, device="cuda:0")
stream = torch.cuda.ExternalStream(machine_stream(tm), device="cuda:0")
ms = []
for r in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _capi.check(_capi.lib().tmg_class_sums_device(tm.handle, test.handle, T.PREDICT, sums.data_ptr()))
    e1.record(stream)
    torch.cuda.synchronize()
    if r:
        ms.append(e0.elapsed_time(e1))
gpu_ms = min(ms)
pred = T.predict_all(tm, test)
evals = 10 * n * qt * 2 * 784
out = {"clauses_per_class": n, "epochs_trained": epochs, "test_rows": qt, "gpu_ms": gpu_ms,
       "gpu_rows_per_s": qt / (gpu_ms * 1e-3), "gpu_clause_literal_evals_per_s": evals / (gpu_ms * 1e-3),
       "gpu_accuracy": float((pred == d.test_y).mean())}
os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
path = os.path.join(os.environ.get("TMPDIR", "/tmp"), f"mnist{n}.model")  # ~100 MB of text
model_io.save_model_file(path, tm)
ref = os.path.join(REPO, "oracle", "_ref", "ref_driver")
if os.path.exists(ref) and ref_rows > 0:
    r = json.loads(subprocess.run([ref, "predict", path, "--data", "mnist", "--q", str(q), "--qtest", str(qt),
                                   "--qtest-use", str(ref_rows), "--data-seed", str(seed)],
                                  check=True, capture_output=True, text=True).stdout)
    ref_pred = np.load(path + ".ref_pred.npy")
    out["ref"] = r
    out["predictions_identical"] = bool(np.array_equal(ref_pred, pred[:ref_rows]))
    out["speedup_rows_per_s"] = out["gpu_rows_per_s"] / r["rows_per_s"]
print(json.dumps(out))
