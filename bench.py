#!/usr/bin/env python3
"""Benchmark of the asynchronous clause-parallel Tsetlin Machine on B200.

Workload (BASELINE.json configs[1]): MNIST-shaped synthetic data, 784 bits x
10 classes, 2000 clauses per class per GPU, T=50, s=10, 8-bit automata
(N=128), q=60,000 training examples (synthetic, generated in-process).

One step = one asynchronous training epoch (Algorithm 1) of a FRESH machine
(reset to counters=N, tallies and previous outputs 0, epoch index 0) over all
q examples — the most expensive epoch, and identical work every step.

  value : clause-literal evals/s = m * n_total * q * 2o / step time, inputs
          resident in HBM, CUDA events on the engine's stream, max over ranks
  e2e   : the same through the C ABI with HOST buffers: per step the pinned
          host bits/labels are copied in (tmg_pool_create), the machine is
          reset, the epoch runs, the per-class feedback-event report is read
          back.
Multi-GPU (torchrun): weak scaling in clauses — every rank owns 2000 clauses
per class (global n = 2000 * world). Default exchange "ipc": the engine's own
communicator (tmg_comm_create_ipc, handles all-gathered once through
torch.distributed) attached to the rank's shard; tmg_train_epoch runs the
rank's epoch as one launch and exchanges the tally deltas beside it, each rank
pulling the others' snapshots over CUDA IPC / NVLink with the copy engines
(paper_2009_04861_b200/csrc/group.cu). "comm" does the same sums with NCCL. Alternatives: "peer" (every tally
change also RED-added into the other ranks' replicas over CUDA IPC / NVLink
by the training kernels), "overlapped"/"sync" (the same windows driven from
Python with torch.distributed, paper_2009_04861_b200/distributed.py).

--impl reference times the UNMODIFIED reference (oracle/_ref/ref_driver, the
reference sources compiled with their own Release flags) on the host cores:
train_epoch_parallel with all hardware threads, fresh epoch 0 per step, on a
bounded q-prefix sample of the same data.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

O_FEAT, M_CLS, N_CLAUSES, MARGIN, SPEC, STATE_N = 784, 10, 2000, 50, 10.0, 128
Q_TRAIN, Q_TEST = 60000, 10000
DATA_SEED, TM_SEED = 2009, 42
REF_DRIVER = os.path.join(REPO, "oracle", "_ref", "ref_driver")
METRIC = "clause-literal evals/s (async training epoch, MNIST-shaped 784b x 10c x 2000 clauses)"
UNIT = "clause-literal evals/s"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(
        os.environ.get("LOCAL_RANK", 0))


# ----------------------------------------------------------------- clocks ---
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.samples, self.proc = device, [], None

    def start(self):
        if not shutil.which("nvidia-smi"):
            return
        self.proc = subprocess.Popen(
            ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
             "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([f.strip() for f in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(s[0]) for s in self.samples if len(s) >= 7 and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 7 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples if len(s) >= 7 for k in range(4)
                          if s[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------- reference arm ---
def ref_driver_run(q_use: int, steps: int, workers: int) -> list:
    args = [REF_DRIVER, "train", "--data", "mnist", "--q", str(q_use), "--qtest", "0", "--clauses",
            str(N_CLAUSES), "--T", str(MARGIN), "--s", str(SPEC), "--N", str(STATE_N), "--epochs",
            str(steps), "--workers", str(workers), "--seed", str(TM_SEED), "--data-seed", str(DATA_SEED),
            "--eval", "0", "--fresh", "1"]
    out = subprocess.run(args, check=True, capture_output=True, text=True).stdout
    return [json.loads(l) for l in out.splitlines() if l.strip()]


def cpu_sample_size(cores: int, budget_s: float) -> int:
    # ~17 examples/s per core at this shape on epoch 0; calibrate.
    probe_q = 200
    rows = ref_driver_run(probe_q, 1, cores)
    per_ex = rows[0]["seconds"] / probe_q
    return int(max(200, min(Q_TRAIN, budget_s / max(per_ex, 1e-6))))


def evals(q: int, n_total: int) -> float:
    return float(M_CLS) * n_total * q * 2 * O_FEAT


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    if not os.path.exists(REF_DRIVER):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_driver not built"}))
        return 0
    cores = os.cpu_count() or 1
    per_step_budget = max(3.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    q_use = cpu_sample_size(cores, per_step_budget)
    rows = ref_driver_run(q_use, args.warmup + args.steps, cores)[args.warmup:]
    secs = [r["seconds"] for r in rows]
    t = max(statistics.mean(secs), 1e-9)
    value = evals(q_use, N_CLAUSES) / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": "mnist-784b-10c-2000cl fresh epoch 0", "q_sample": q_use, "q_full": Q_TRAIN,
                   "clauses_per_class": N_CLAUSES, "T": MARGIN, "s": SPEC, "state_bits": 8},
        "examples_per_s": q_use / t,
        "feedback_events_per_step": statistics.mean(r["feedback_events"] for r in rows),
        "feedback_events_per_s": statistics.mean(r["feedback_events"] for r in rows) / t,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"fresh-model epoch 0 on the first {q_use} of {Q_TRAIN} training rows, "
                                   f"train_epoch_parallel(workers={cores})"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------- ours ---
def algorithmic_ops(steps_per_epoch: int, events: int, type1: int) -> float:
    """SURVEY.md §8(d) cost model (fixed up front): gate = 1 draw (~15 int ops)
    + 3; per event 2*ceil(2o/32) LOP3 of evaluation; Type I = 2o TA updates of
    (1 draw + 3); Type II = 2o TA updates of 3."""
    L = 2 * O_FEAT
    w32 = (L + 31) // 32
    return 18.0 * steps_per_epoch + events * 2.0 * w32 + type1 * L * 18.0 + (events - type1) * L * 3.0


def inference_line(args, tm, d, local, stream, clk=None):
    import numpy as np
    import torch

    import ctypes as C

    import paper_2009_04861_b200 as T
    from paper_2009_04861_b200 import _capi, model_io

    tx = torch.from_numpy(d.test_x).to(f"cuda:{local}")
    ty = torch.from_numpy(d.test_y).to(f"cuda:{local}")
    torch.cuda.synchronize()
    test = T.ExamplePool.from_device(O_FEAT, tx.data_ptr(), ty.data_ptr(), Q_TEST, M_CLS, device=local,
                                     labels_host=d.test_y)
    sums = torch.zeros(Q_TEST * M_CLS, dtype=torch.int32, device=f"cuda:{local}")
    ms = []
    for r in range(args.warmup + args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _capi.check(_capi.lib().tmg_class_sums_device(tm.handle, test.handle, T.PREDICT, sums.data_ptr()))
        e1.record(stream)
        torch.cuda.synchronize()
        if r >= args.warmup:
            ms.append(e0.elapsed_time(e1))
    t = statistics.mean(ms)
    kms = []  # the class-sum kernel alone (events inside the library around its launch)
    for _ in range(3):
        _capi.check(_capi.lib().tmg_class_sums_device(tm.handle, test.handle, T.PREDICT, sums.data_ptr()))
        v = C.c_float()
        _capi.check(_capi.lib().tmg_last_eval_kernel_ms(tm.handle, C.byref(v)))
        kms.append(v.value)
    kernel_ms = statistics.mean(kms)
    pred = T.predict_all(tm, test)
    evals_per_s = M_CLS * N_CLAUSES * Q_TEST * 2 * O_FEAT / (t * 1e-3)
    out = {"metric": "clause-literal evals/s (predict, class sums of the test rows)", "value": evals_per_s,
           "unit": "clause-literal evals/s", "rows_per_s": Q_TEST / (t * 1e-3), "ms": t, "rows": Q_TEST,
           "kernel": "eval_bits_kernel<0>", "model": "state after the last timed epoch",
           "test_accuracy": float((pred == d.test_y).mean()),
           "kernel_ms": kernel_ms,
           "roofline": roofline_record("eval_bits_ncu.json", kernel_ms * 1e-3, clk, "eval_bits_kernel<0>", t,
                                       extra={"timing_note": "kernel_ms: CUDA events around the eval_bits_kernel "
                                                             "launch alone (tmg_last_eval_kernel_ms); the call "
                                                             "(`ms`) adds the sums memset"})}
    if not args.no_cpu and os.path.exists(REF_DRIVER):
        import tempfile
        rows = 500
        with tempfile.TemporaryDirectory() as tmp:
            path = os.path.join(tmp, "bench.model")
            model_io.save_model_file(path, tm)
            r = json.loads(subprocess.run(
                [REF_DRIVER, "predict", path, "--data", "mnist", "--q", str(Q_TRAIN), "--qtest", str(Q_TEST),
                 "--qtest-use", str(rows), "--data-seed", str(DATA_SEED)],
                check=True, capture_output=True, text=True).stdout)
            same = bool(np.array_equal(np.load(path + ".ref_pred.npy"), pred[:rows]))
        out["cpu_baseline"] = {"value": M_CLS * N_CLAUSES * rows * 2 * O_FEAT / r["seconds"],
                               "unit": "clause-literal evals/s", "rows_per_s": r["rows_per_s"], "cores": 1,
                               "kind": "reference",
                               "sample": f"predict_all (single-threaded by construction, trainer.cpp:272-279) "
                                         f"on the first {rows} test rows, same model file"}
        out["predictions_identical"] = same
    return out


def other_configs(local):
    """BASELINE.json configs[2] and [3] on this GPU: one fresh async epoch
    (after one untimed one) of the FMNIST- and IMDb-shaped workloads,
    device time on the engine stream. Reported beside the headline; the
    parity tests cover their accuracy."""
    import paper_2009_04861_b200 as T
    from paper_2009_04861_b200 import synth
    import torch
    from paper_2009_04861_b200 import _capi
    from paper_2009_04861_b200.tsetlin import machine_stream
    out = []
    for kind, q, qt, n, T_, s_, seed in (("fmnist", 60000, 10000, 8000, 100, 15.0, 2352),
                                         ("imdb", 25000, 25000, 10000, 100, 15.0, 10000)):
        d = synth.make(kind, q, qt, seed)
        tm = T.MultiClassTM(T.TMConfig(clauses=n, margin=T_, specificity=s_, seed=TM_SEED), d.features, d.classes,
                            device=local)
        pool = T.ExamplePool(d.features, d.train_x, d.train_y, d.classes, device=local)
        for r in range(2):
            tm.reset()
            pool.reset_tallies()
            rep = T.train_epoch_parallel(tm, pool, 1, 0)
        t = rep.device_seconds
        # predict: class sums of the test rows on the trained state (device time)
        test = T.ExamplePool(d.features, d.test_x, d.test_y, d.classes, device=local)
        sums = torch.zeros(qt * d.classes, dtype=torch.int32, device=f"cuda:{local}")
        stream = torch.cuda.ExternalStream(machine_stream(tm), device=f"cuda:{local}")
        pms = []
        for r in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _capi.check(_capi.lib().tmg_class_sums_device(tm.handle, test.handle, T.PREDICT, sums.data_ptr()))
            e1.record(stream)
            torch.cuda.synchronize()
            if r:
                pms.append(e0.elapsed_time(e1))
        rec = {"workload": f"{kind} {d.features}b x {d.classes}c x {n} clauses, q={q}, fresh epoch 0",
               "ms_per_epoch": t * 1e3, "examples_per_s": q / t,
               "clause_literal_evals_per_s": d.classes * n * q * 2.0 * d.features / t,
               "feedback_events": rep.total_feedback_events(),
               "predict_test_rows": qt, "predict_ms": min(pms),
               "test_accuracy_after_epoch0": T.evaluate_accuracy(tm, test)}
        # the committed ncu capture of this shape's training kernel (same
        # command shape, tools/gpu_final_r2.sh): pipe use and DRAM per launch
        prof = os.path.join(REPO, "profiles", {"fmnist": "r2w_fmnist_async.json", "imdb": "r2w_imdb_smem.json"}[kind])
        if os.path.exists(prof):
            pj = json.load(open(prof))
            rec["ncu"] = {k: pj.get(k) for k in ("kernel", "duration_ms", "pipe_alu_pct", "issue_active_pct",
                                                  "dram_bytes_per_launch", "registers_per_thread",
                                                  "occupancy_achieved_pct")}
            rec["ncu"]["source"] = os.path.relpath(prof, REPO)
        out.append(rec)
        del tm, pool, test
    return out


def sharded_line(d, local) -> dict:
    """The N > 1 machinery on this one GPU: the bench epoch
    through one-rank communicators — CUDA IPC (the N-GPU default) and NCCL —
    (the code path of every rank of the N-GPU run: streaming tally exchange,
    event all-reduce) against the plain machine, and a two-shard machine on this GPU (peer-memory sums) against
    one machine of the same clause count. Fresh epoch 0, best of 3."""
    import paper_2009_04861_b200 as T
    pool = T.ExamplePool(O_FEAT, d.train_x, d.train_y, M_CLS, device=local)

    def best(tm):
        out = []
        for _ in range(4):
            tm.reset()
            pool.reset_tallies()
            out.append(T.train_epoch_parallel(tm, pool, 1, 0).seconds * 1e3)
        return min(out[1:])

    cfg = T.TMConfig(clauses=N_CLAUSES, margin=MARGIN, specificity=SPEC, state_depth=STATE_N, seed=TM_SEED)
    out = {"plain_ms": best(T.MultiClassTM(cfg, O_FEAT, M_CLS, device=local))}
    ok, why = T.nccl_available()
    if ok:
        comm = T.Comm(T.Comm.unique_id(), 1, 0, local)
        tm = T.MultiClassTM(cfg, O_FEAT, M_CLS, device=local, clause_range=(0, N_CLAUSES))
        tm.attach_comm(comm)
        out["one_rank_comm_ms"] = best(tm)
        out["one_rank_comm_overhead"] = out["one_rank_comm_ms"] / out["plain_ms"]
        tm.attach_comm(None)
        del tm, comm
    else:
        out["nccl"] = why
    ipc = T.Comm.ipc(1, 0, local, Q_TRAIN * M_CLS, lambda b: [b])  # the N-GPU default's code path
    tm = T.MultiClassTM(cfg, O_FEAT, M_CLS, device=local, clause_range=(0, N_CLAUSES))
    tm.attach_comm(ipc)
    out["one_rank_ipc_ms"] = best(tm)
    out["one_rank_ipc_overhead"] = out["one_rank_ipc_ms"] / out["plain_ms"]
    tm.attach_comm(None)
    del tm, ipc
    cfg2 = T.TMConfig(clauses=2 * N_CLAUSES, margin=MARGIN, specificity=SPEC, state_depth=STATE_N, seed=TM_SEED)
    out["plain_2x_clauses_ms"] = best(T.MultiClassTM(cfg2, O_FEAT, M_CLS, device=local))
    out["two_shards_one_gpu_ms"] = best(T.MultiClassTM(cfg2, O_FEAT, M_CLS, devices=[local, local]))
    out["two_shards_overhead"] = out["two_shards_one_gpu_ms"] / out["plain_2x_clauses_ms"]
    return out


def sequential_line(local, with_ref: bool) -> dict:
    """train_epoch_sequential, the reference's classic
    trainer replayed bit-exactly on the GPU (gate scan with xoshiro jump-ahead,
    gated clauses applied grid-wide), fresh machine, epoch 0, on the first
    500 MNIST-shaped rows; the reference's own sequential trainer (one thread
    by construction) on the same rows beside it. Equal feedback-event counts
    are the bit-exactness check visible here (the tests compare states)."""
    import paper_2009_04861_b200 as T
    from paper_2009_04861_b200 import synth
    q = 500
    d = synth.make("mnist", q, 0, DATA_SEED)
    tm = T.MultiClassTM(T.TMConfig(clauses=N_CLAUSES, margin=MARGIN, specificity=SPEC, seed=TM_SEED), O_FEAT,
                        M_CLS, device=local)
    pool = T.ExamplePool(O_FEAT, d.train_x, d.train_y, M_CLS, device=local)
    T.train_epoch_sequential(tm, pool, 0)  # warm-up (matrices, scratch)
    tm.reset()
    pool.reset_tallies()
    rep = T.train_epoch_sequential(tm, pool, 0)
    line = {"workload": f"mnist-784b-10c-{N_CLAUSES}cl train_epoch_sequential, fresh epoch 0, first {q} rows",
            "seconds": rep.seconds, "examples_per_s": q / rep.seconds,
            "feedback_events": rep.total_feedback_events()}
    if with_ref and os.path.exists(REF_DRIVER):
        args = [REF_DRIVER, "train", "--data", "mnist", "--mode", "seq", "--q", str(q), "--qtest", "0", "--clauses",
                str(N_CLAUSES), "--T", str(MARGIN), "--s", str(SPEC), "--N", str(STATE_N), "--epochs", "1",
                "--seed", str(TM_SEED), "--data-seed", str(DATA_SEED), "--eval", "0", "--fresh", "1"]
        r = json.loads(subprocess.run(args, check=True, capture_output=True, text=True).stdout.splitlines()[-1])
        line["reference"] = {"seconds": r["seconds"], "examples_per_s": q / r["seconds"], "cores": 1,
                             "feedback_events": r["feedback_events"], "kind": "reference"}
        line["speedup_vs_reference"] = r["seconds"] / rep.seconds
        line["events_identical"] = r["feedback_events"] == rep.total_feedback_events()
    return line


SM_COUNT, SCHEDULERS_PER_SM = 148, 4


def same_q_record(d, local, q_use: int, ref_row: dict, line: dict) -> dict:
    """Like-for-like with the reference's sample: the GPU's fresh epoch 0 on
    the SAME first q_use training rows (examples/s and feedback events/s of
    both), beside the full-q events/s ratio. Per-example cost depends on q
    (the tallies of a longer epoch saturate later), so the events-normalised
    ratio is the fair one for the headline."""
    import paper_2009_04861_b200 as T
    tm = T.MultiClassTM(T.TMConfig(clauses=N_CLAUSES, margin=MARGIN, specificity=SPEC, state_depth=STATE_N,
                                   seed=TM_SEED), O_FEAT, M_CLS, device=local)
    pool = T.ExamplePool(O_FEAT, d.train_x[:q_use], d.train_y[:q_use], M_CLS, device=local)
    secs, ev = [], []
    for _ in range(4):  # first is warm-up
        tm.reset()
        pool.reset_tallies()
        rep = T.train_epoch_parallel(tm, pool, 1, 0)
        secs.append(rep.device_seconds)
        ev.append(rep.total_feedback_events())
    g_s, g_ev = statistics.mean(secs[1:]), statistics.mean(ev[1:])
    r_s, r_ev = ref_row["seconds"], ref_row["feedback_events"]
    return {"q": q_use, "gpu_ms": g_s * 1e3, "gpu_examples_per_s": q_use / g_s,
            "gpu_feedback_events_per_s": g_ev / g_s, "gpu_feedback_events": g_ev,
            "ref_examples_per_s": q_use / r_s, "ref_feedback_events_per_s": r_ev / r_s, "ref_feedback_events": r_ev,
            "examples_ratio_same_q": (q_use / g_s) / (q_use / r_s),
            "events_ratio_same_q": (g_ev / g_s) / (r_ev / r_s),
            "events_ratio_full_q": line["feedback_events_per_s"] / (r_ev / r_s),
            "examples_ratio_full_q_vs_prefix": line["examples_per_s"] / (q_use / r_s)}


def time_to_accuracy(d, local, epochs: int = 5) -> dict:
    """Test accuracy after every asynchronous epoch (q = 60 000, 10 000 test
    rows, seed 42) and the device time to reach the reference's mean final
    accuracy (tests/golden/accuracy_ref.json "mnist_q60000": 5 seeds x 3
    epochs of the compiled reference, train_epoch_parallel on all 8 threads
    of the build container; its epoch seconds are that machine's)."""
    import paper_2009_04861_b200 as T
    allref = json.load(open(os.path.join(REPO, "tests", "golden", "accuracy_ref.json")))
    ref = allref.get("mnist_q60000")
    tm = T.MultiClassTM(T.TMConfig(clauses=N_CLAUSES, margin=MARGIN, specificity=SPEC, state_depth=STATE_N,
                                   seed=TM_SEED), O_FEAT, M_CLS, device=local)
    pool = T.ExamplePool(O_FEAT, d.train_x, d.train_y, M_CLS, device=local)
    test = T.ExamplePool(O_FEAT, d.test_x, d.test_y, M_CLS, device=local)
    acc, secs = [], []
    for e in range(epochs):
        rep = T.train_epoch_parallel(tm, pool, 1, e)
        secs.append(rep.device_seconds)
        acc.append(T.evaluate_accuracy(tm, test))
    out = {"gpu_accuracy_per_epoch": [round(a, 4) for a in acc], "gpu_epoch_ms": [round(v * 1e3, 2) for v in secs]}
    if ref:
        seeds = sorted(ref["per_seed"])
        ref_acc = [statistics.mean(ref["per_seed"][k][e] for k in seeds) for e in range(len(ref["per_seed"][seeds[0]]))]
        ref_s = [statistics.mean(ref["epoch_seconds"][k][e] for k in seeds) for e in range(len(ref_acc))]
        target = ref_acc[-1]
        hit = next((e for e, a in enumerate(acc) if a >= target), None)
        out.update({"target": round(target, 4), "target_source": "reference mean final accuracy, 5 seeds, "
                                                                 f"{len(ref_acc)} epochs (W={ref['workers']})",
                    "reference_accuracy_per_epoch": [round(a, 4) for a in ref_acc],
                    "reference_epoch_s": [round(v, 1) for v in ref_s],
                    "reference_seconds_to_target": round(sum(ref_s), 1),
                    "gpu_epochs_to_target": None if hit is None else hit + 1,
                    "gpu_seconds_to_target": None if hit is None else sum(secs[:hit + 1]),
                    "speedup_to_target": None if hit is None else sum(ref_s) / sum(secs[:hit + 1])})
        by_w = {}
        for key in ("mnist_q60000", "mnist_q60000_w4", "mnist_q60000_w2", "mnist_q60000_w1"):
            if key in allref:
                v = allref[key]
                ks = sorted(v["per_seed"])
                by_w[f"W={v['workers']}"] = {
                    "seeds": len(ks),
                    "accuracy_per_epoch": [round(statistics.mean(v["per_seed"][k][e] for k in ks), 4)
                                           for e in range(len(v["per_seed"][ks[0]]))],
                    "epoch_s": [round(statistics.mean(v["epoch_seconds"][k][e] for k in ks), 1)
                                for e in range(len(v["per_seed"][ks[0]]))]}
        out["reference_by_workers"] = by_w
    return out


def roofline_record(profile: str, kernel_s: float, clk, kernel: str, step_ms: float, effective=None, extra=None):
    """Issue-bound roofline of one kernel: ncu's executed warp instructions of
    this workload (profiles/<profile>, an ncu --set full capture of the same
    command) / the kernel's live duration, vs the issue peak at the measured
    SM clock. frac is a hardware fraction (<= 1); the ncu pipe and memory
    utilisations of the same capture ride along."""
    path = os.path.join(REPO, "profiles", profile)
    prof = json.load(open(path)) if os.path.exists(path) else {}
    mhz = (clk or {}).get("sm_mhz") or (clk or {}).get("sm_max_mhz") or 1965.0
    peak = SM_COUNT * SCHEDULERS_PER_SM * 32 * mhz * 1e6  # thread-instructions/s
    instr = prof.get("warp_instructions")
    achieved = instr * 32 / kernel_s if instr else None
    rec = {"bound": "int-issue", "unit": "Tops/s (thread instructions)",
           "achieved": achieved / 1e12 if achieved else None, "peak": peak / 1e12,
           "frac": achieved / peak if achieved else None,
           "traffic": prof.get("dram_bytes_per_launch"),
           "kernel": kernel, "kernel_ms": kernel_s * 1e3, "kernel_share_of_step": kernel_s * 1e3 / step_ms,
           "instructions_per_launch": instr, "ncu_duration_ms": prof.get("duration_ms"),
           "ncu": {k: prof.get(k) for k in ("pipe_alu_pct", "pipe_fma_pct", "pipe_fmaheavy_pct", "pipe_lsu_inst_pct",
                                            "issue_active_pct", "l1tex_throughput_pct", "l2_throughput_pct",
                                            "occupancy_achieved_pct", "source") if k in prof},
           "peak_source": f"issue peak {SM_COUNT} SMs x {SCHEDULERS_PER_SM} schedulers x 32 lanes at the sampled "
                          f"SM clock ({mhz:.0f} MHz); MEASURED_PEAKS.json has no integer figure",
           "profile": f"profiles/{profile}"}
    if effective is not None:
        rec["effective_frac"] = effective
    rec.update(extra or {})
    return rec


def run_ours(args):
    import numpy as np
    import torch

    import paper_2009_04861_b200 as T
    from paper_2009_04861_b200 import distributed as D
    from paper_2009_04861_b200 import synth
    from paper_2009_04861_b200.tsetlin import int_peak, kernel_launches, machine_stream

    rank, world, local = dist_env()
    if args.share_device:  # protocol test: every rank on cuda:0 (gloo; NCCL rejects duplicate GPUs)
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(args.dist_backend)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    d = synth.make("mnist", Q_TRAIN, Q_TEST, DATA_SEED)
    n_total = N_CLAUSES * world
    jb, je = D.shard_range(n_total, rank, world)
    cfg = T.TMConfig(clauses=n_total, margin=MARGIN, specificity=SPEC, state_depth=STATE_N, seed=TM_SEED)
    tm = T.MultiClassTM(cfg, O_FEAT, M_CLS, device=local, clause_range=(jb, je) if world > 1 else None)
    # Resident inputs: bits/labels already in HBM (torch allocations), packed on device.
    d_bits = torch.from_numpy(d.train_x).to(f"cuda:{local}")
    d_lab = torch.from_numpy(d.train_y).to(f"cuda:{local}")
    pool = T.ExamplePool.from_device(O_FEAT, d_bits.data_ptr(), d_lab.data_ptr(), Q_TRAIN, M_CLS, device=local,
                                     labels_host=d.train_y)
    stream = torch.cuda.ExternalStream(machine_stream(tm), device=f"cuda:{local}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=f"cuda:{local}")  # > 126 MB L2
    allreduce = D.nccl_allreduce(local) if world > 1 else None
    windows = args.windows
    exchange, exchange_note = (args.exchange if world > 1 else "none"), None
    comm = None
    if exchange == "comm" and (args.share_device or args.dist_backend != "nccl"):
        exchange, exchange_note = "ipc", "NCCL needs one GPU per rank; one-device protocol test over CUDA IPC"
    if exchange == "comm":  # the library's NCCL communicator, streaming exchange inside tmg_train_epoch
        uid = [T.Comm.unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(uid, src=0)
        comm = T.Comm(uid[0], world, rank, local)
        tm.attach_comm(comm)
        tm.set_windows(windows)
    elif exchange == "ipc":  # the same exchange, snapshots pulled over CUDA IPC by the copy engines

        def allgather(b):
            out = [None] * world
            torch.distributed.all_gather_object(out, b)
            return out

        comm = T.Comm.ipc(world, rank, local, Q_TRAIN * M_CLS, allgather)
        tm.attach_comm(comm)
        tm.set_windows(windows)
    if exchange == "peer":  # tally replicas over peer memory; NCCL windows if P2P is unavailable
        try:
            D.attach_peer_tallies(pool)
        except Exception as e:  # noqa: BLE001 - any IPC failure falls back, and is reported
            exchange, exchange_note = "overlapped", f"peer memory unavailable ({e}); fell back"
        ok = torch.tensor([1 if exchange == "peer" else 0], device=f"cuda:{local}")
        torch.distributed.all_reduce(ok, op=torch.distributed.ReduceOp.MIN)
        if int(ok.item()) == 0 and exchange == "peer":
            D.detach_peer_tallies(pool)
            exchange, exchange_note = "overlapped", "a peer could not map the replicas; fell back"

    def one_epoch(p):
        tm.reset()
        p.reset_tallies()
        if world == 1 or exchange in ("comm", "ipc"):
            rep = T.train_epoch_parallel(tm, p, 1, 0)
            return rep.feedback_events, rep.type_i_events, (rep.device_seconds if world == 1 else None)
        if exchange == "peer":
            ev = D.train_epoch_peer(tm, p, 0)
        elif exchange == "overlapped":
            ev = D.train_epoch_overlapped(tm, p, 0, windows)
        else:
            ev = D.train_epoch_windows(D.GpuShardEngine(tm, p), 0, windows, allreduce)
        return ev, None, None

    # ---- integer-pipe peak (roofline denominator), measured on this GPU
    lop3_peak, mixed_peak = int_peak(local)

    # ---- warm-up
    for _ in range(args.warmup):
        one_epoch(pool)
    torch.cuda.synchronize()

    # ---- timed: inputs resident
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
    step_ms, kern_s, events, type1 = [], [], [], []
    launches0 = kernel_launches()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ev, t1, ks = one_epoch(pool)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        step_ms.append(max_over_ranks(e0.elapsed_time(e1)))
        events.append(sum(ev))
        if t1 is not None:
            type1.append(sum(t1))
        if ks is not None:
            kern_s.append(ks)
    launches = kernel_launches() - launches0
    clk = clocks.stop() if clocks else None

    # ---- e2e: host buffers through the C ABI, copies inside the timed region
    host_bits = torch.from_numpy(d.train_x).pin_memory().numpy()
    host_lab = torch.from_numpy(d.train_y).pin_memory().numpy()
    e2e_ms, e2e_phases = [], []
    for it in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        p2 = T.ExamplePool(O_FEAT, host_bits, host_lab, M_CLS, device=local)
        if exchange == "peer":
            D.attach_peer_tallies(p2)
        t1 = time.perf_counter()
        ev, _, _ = one_epoch(p2)
        _ = [int(v) for v in ev]  # per-class report read back to the host
        t2 = time.perf_counter()
        if exchange == "peer":
            D.detach_peer_tallies(p2)
            barrier()
        del p2
        torch.cuda.synchronize()
        barrier()
        t3 = time.perf_counter()
        dt = max_over_ranks((t3 - t0) * 1e3)
        if it >= args.warmup:  # the same W untimed warm-up steps as the resident arm
            e2e_ms.append(dt)
            e2e_phases.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3))

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0

    ms = statistics.mean(step_ms)
    value = evals(Q_TRAIN, n_total) / (ms * 1e-3)
    e2e_val = evals(Q_TRAIN, n_total) / (statistics.mean(e2e_ms) * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": "mnist-784b-10c-2000cl fresh epoch 0", "q": Q_TRAIN,
                   "clauses_per_class_per_gpu": N_CLAUSES, "clauses_per_class_total": n_total,
                   "T": MARGIN, "s": SPEC, "state_bits": 8, "parallelism": f"clause-shard{world}",
                   "windows": windows if world > 1 and exchange != "peer" else 1,
                   "exchange": exchange,
                   **({"exchange_note": exchange_note} if exchange_note else {}),
                   "l2": "flushed (256 MB write) between timed steps; working set (prev bits 150 MB) > L2"},
        "examples_per_s": Q_TRAIN / (ms * 1e-3),
        "feedback_events_per_step": statistics.mean(events),
        "feedback_events_per_s": statistics.mean(events) / (ms * 1e-3),
        "ta_updates_per_s": statistics.mean(events) * 2.0 * O_FEAT / (ms * 1e-3),  # 2o per event
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    # ---- roofline of the dominant kernel (train_async): integer issue bound.
    # Hardware fraction: the kernel's executed warp instructions per launch
    # (ncu, committed profile of this exact workload) over its live CUDA-event
    # time, against the SM issue peak (148 SMs x 4 schedulers x 1 warp
    # instruction per cycle) at the SM clock sampled during the timed region.
    if kern_s:
        k = statistics.mean(kern_s)
        line["roofline"] = roofline_record(
            "train_async_ncu.json", k, clk, "train_async_kernel<1,8,P2>", ms,
            effective=algorithmic_ops(M_CLS * N_CLAUSES * Q_TRAIN, int(statistics.mean(events)),
                                      int(statistics.mean(type1))) / k / mixed_peak,
            extra={"effective_note": "SURVEY.md 8(d) ops model (gate 18, eval 2*ceil(2o/32), TypeI 2o*18, "
                                     "TypeII 2o*3) / kernel time / measured LOP3+IMAD peak "
                                     f"{mixed_peak / 1e12:.2f} Tops/s (LOP3-only {lop3_peak / 1e12:.2f}); "
                                     ">1 because the alias sampler draws one 32-bit word per 8 literals"})
    line["e2e"] = {"value": e2e_val, "unit": UNIT, "ms_per_step": statistics.mean(e2e_ms),
                   "ms_all": [round(v, 3) for v in e2e_ms],
                   "phases_ms": {k: round(statistics.mean(ph[n] for ph in e2e_phases), 3)
                                 for n, k in enumerate(("pool_h2d_pack", "epoch_and_report", "pool_free"))},
                   "h2d_bytes_per_step": int(host_bits.nbytes + host_lab.nbytes + 4 * Q_TRAIN),
                   "d2h_bytes_per_step": int(8 * M_CLS * 2)}
    # ---- inference on the state the last timed epoch left (class sums of the
    # 10 000 test rows; K1 eval kernel, CUDA events on the engine stream),
    # beside the reference's single-threaded predict_all on the SAME model
    # file for a bounded row sample, predictions compared row for row.
    if world == 1:
        line["inference"] = inference_line(args, tm, d, local, stream, clk)
        if not args.no_other_configs:
            line["other_configs"] = other_configs(local)
            line["sequential_trainer"] = sequential_line(local, not args.no_cpu)
            line["sharded_path"] = sharded_line(d, local)
    # ---- CPU reference beside it (rank 0, N=1 only)
    if world == 1 and not args.no_cpu and os.path.exists(REF_DRIVER):
        cores = os.cpu_count() or 1
        q_use = cpu_sample_size(cores, 15.0)
        rows = ref_driver_run(q_use, 1, cores)
        t = rows[0]["seconds"]
        line["cpu_baseline"] = {"value": evals(q_use, N_CLAUSES) / t, "unit": UNIT, "cores": cores,
                                "kind": "reference", "examples_per_s": q_use / t,
                                "feedback_events_per_s": rows[0]["feedback_events"] / t,
                                "sample": f"fresh-model epoch 0 on the first {q_use} of {Q_TRAIN} rows, "
                                          f"reference train_epoch_parallel(workers={cores}), "
                                          f"{rows[0]['feedback_events']} feedback events"}
        line["same_q"] = same_q_record(d, local, q_use, rows[0], line)
    if world == 1 and not args.no_other_configs:
        line["time_to_accuracy"] = time_to_accuracy(d, local)
    print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--windows", type=int, default=16, help="tally all-reduce windows per epoch (N>1; 16 costs ~2%% on one GPU, tools/window_cost.py)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-other-configs", action="store_true", help="skip the FMNIST/IMDb side measurements")
    ap.add_argument("--dist-backend", default="nccl", help="torch.distributed backend for N>1 (tests: gloo)")
    ap.add_argument("--exchange", choices=["ipc", "comm", "peer", "overlapped", "sync"], default="ipc",
                    help="N>1 tally exchange: the engine's streaming exchange inside tmg_train_epoch with the "
                         "ranks' snapshots pulled over CUDA IPC by the copy engines (default) or summed by an "
                         "NCCL communicator; replicas updated by the training kernels over peer memory "
                         "(NVLink); windowed all-reduce driven from Python, overlapped or host-synchronous")
    ap.add_argument("--share-device", action="store_true",
                    help="run every rank on cuda:0 (one-GPU test of the N>1 protocol; not a measurement)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
