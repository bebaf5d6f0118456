"""Clause-count timing sweep with the reference's CSV schema (SURVEY.md §8(f)
row f4; reference: proj/src/bench.cpp:45-142, bench.hpp:28-58), so GPU rows
line up with the CPU reference's `tm bench` output.

Modes: "seq" = train_epoch_sequential (GPU mirror), "par" =
train_epoch_parallel in TMG_MODE_AUTO, like the C++ facade (the asynchronous
all-clause GPU trainer; the bit-exact one-worker replay when workers == 1 and
TSETLIN_DETERMINISTIC=1). `seconds` is the epoch
only (EpochReport.seconds); the metric is test accuracy (or MAE for
regression) after each measured epoch.
"""
from __future__ import annotations

import csv
import io
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import tsetlin as T


@dataclass
class BenchRecord:  # bench.hpp:28-36
    mode: str
    workers: int
    clauses: int
    epoch: int
    seconds: float
    metric_name: str
    metric_value: float


@dataclass
class BenchOptions:  # bench.hpp:38-45
    clause_counts: Sequence[int] = field(default_factory=list)
    modes: Sequence[str] = ("seq",)
    warmup_epochs: int = 1
    measured_epochs: int = 3
    workers: int = 0  # 0 = the async GPU trainer
    regression: bool = False


def bench_sweep(train_x, train_y, test_x, test_y, base: T.TMConfig, options: BenchOptions) -> List[BenchRecord]:
    """bench_sweep (bench.cpp:45-118) on the GPU."""
    if not options.clause_counts:
        raise ValueError("bench needs at least one clause count")
    for mode in options.modes:
        if mode not in ("seq", "par"):
            raise ValueError("bench mode must be seq or par")
    o = train_x.shape[1]
    workers = options.workers if options.workers > 0 else 64
    records = []
    for mode in options.modes:
        for clauses in options.clause_counts:
            cfg = T.TMConfig(**{**base.__dict__, "clauses": clauses})
            cfg.validate()
            total_epochs = options.warmup_epochs + options.measured_epochs
            if options.regression:
                lo, hi = int(np.min(train_y)), int(np.max(train_y))
                head = T.RegressionHead(cfg, o, lo, hi)
                pool = T.regress_pool(head, train_x, train_y)
                test = T.ExamplePool(o, test_x, np.asarray(test_y, np.int32), 1)
                for e in range(total_epochs):
                    rep = (T.train_epoch_regress_sequential(head, pool, e) if mode == "seq"
                           else T.train_epoch_regress_parallel(head, pool, workers, e, mode=T.MODE_AUTO))
                    if e < options.warmup_epochs:
                        continue
                    v = T.predict_scaled_all(head, test).astype(np.float64)
                    pred = head.y_min + v * (head.y_max - head.y_min) / head.config.margin
                    mae = float(np.mean(np.abs(pred - np.asarray(test_y, np.float64))))
                    records.append(BenchRecord(mode, 1 if mode == "seq" else workers, clauses,
                                               e - options.warmup_epochs, rep.seconds, "mae", mae))
                continue
            classes = max(2, int(max(np.max(train_y), np.max(test_y))) + 1)
            tm = T.MultiClassTM(cfg, o, classes)
            pool = T.ExamplePool(o, train_x, train_y, classes)
            test = T.ExamplePool(o, test_x, test_y, classes)
            for e in range(total_epochs):
                if mode == "seq":
                    rep = T.train_epoch_sequential(tm, pool, e)
                else:
                    rep = T.train_epoch_parallel(tm, pool, workers, e, mode=T.MODE_AUTO)
                if e < options.warmup_epochs:
                    continue
                records.append(BenchRecord(mode, 1 if mode == "seq" else workers, clauses,
                                           e - options.warmup_epochs, rep.seconds, "accuracy",
                                           T.evaluate_accuracy(tm, test)))
    return records


def _g9(v: float) -> str:
    return "%.9g" % v  # format_csv_double, bench.cpp:37-41


def write_bench_csv(records: Sequence[BenchRecord]) -> str:
    """write_bench_csv (bench.cpp:120-127)."""
    out = io.StringIO()
    out.write("mode,workers,clauses,epoch,seconds,metric_name,metric_value\n")
    for r in records:
        out.write(f"{r.mode},{r.workers},{r.clauses},{r.epoch},{_g9(r.seconds)},{r.metric_name},"
                  f"{_g9(r.metric_value)}\n")
    return out.getvalue()


def median_epoch_seconds(records: Sequence[BenchRecord], mode: str, clauses: int) -> float:
    """median_epoch_seconds (bench.cpp:129-142)."""
    s = sorted(r.seconds for r in records if r.mode == mode and r.clauses == clauses)
    if not s:
        raise ValueError("no bench records for requested cell")
    mid = len(s) // 2
    return s[mid] if len(s) % 2 else 0.5 * (s[mid - 1] + s[mid])


def read_bench_csv(text: str) -> List[BenchRecord]:
    rows = list(csv.DictReader(io.StringIO(text)))
    return [BenchRecord(r["mode"], int(r["workers"]), int(r["clauses"]), int(r["epoch"]), float(r["seconds"]),
                        r["metric_name"], float(r["metric_value"])) for r in rows]
