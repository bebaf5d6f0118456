#!/usr/bin/env python3
"""train_epoch_parallel(workers = 1), fresh machine, epoch 0, MNIST shape:
the reference's single-worker trainer (oracle/_ref/ref_driver, one host
thread) beside the GPU's two one-worker modes — TMG_MODE_AUTO's default
(the asynchronous all-clause kernel) and the bit-exact replay selected by
TSETLIN_DETERMINISTIC=1 (TMG_MODE_SYNC_MIRROR).

Usage: python tools/w1_compare.py [q n] ... > profiles/<tag>_w1_compare.jsonl
"""
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_04861_b200 as T  # noqa: E402
from paper_2009_04861_b200 import synth  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "oracle", "_ref", "ref_driver")


def gpu(q, n, mode):
    d = synth.make("mnist", q, 10, 2009)
    tm = T.MultiClassTM(T.TMConfig(clauses=n, margin=50, specificity=10.0, seed=42), 784, 10)
    pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
    t0 = time.perf_counter()
    rep = T.train_epoch_parallel(tm, pool, 1, 0, mode=mode)
    return time.perf_counter() - t0, rep.total_feedback_events()


def main():
    args = [int(a) for a in sys.argv[1:]] or [200, 200, 1000, 2000]
    for q, n in zip(args[::2], args[1::2]):
        row = {"shape": "mnist", "q": q, "clauses_per_class": n, "epoch": 0}
        row["gpu_auto_async_s"], row["gpu_auto_async_events"] = gpu(q, n, T.MODE_ASYNC)
        row["gpu_replay_s"], row["gpu_replay_events"] = gpu(q, n, T.MODE_SYNC_MIRROR)
        if os.path.exists(REF):
            out = subprocess.run([REF, "train", "--data", "mnist", "--q", str(q), "--qtest", "10", "--clauses",
                                  str(n), "--T", "50", "--s", "10", "--epochs", "1", "--workers", "1", "--eval",
                                  "0", "--seed", "42", "--data-seed", "2009"],
                                 check=True, capture_output=True, text=True).stdout
            r = json.loads(out.splitlines()[0])
            row["reference_w1_s"], row["reference_w1_events"] = r["seconds"], r["feedback_events"]
            row["replay_events_equal_reference"] = row["gpu_replay_events"] == r["feedback_events"]
            row["replay_vs_reference"] = r["seconds"] / row["gpu_replay_s"]
            row["auto_vs_reference"] = r["seconds"] / row["gpu_auto_async_s"]
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
