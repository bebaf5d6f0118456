#!/usr/bin/env python3
"""Clause-count sweep (BASELINE.json configs[4]): fresh async epoch-0 time on
MNIST-shaped data vs clauses per class, plus the FMNIST-/IMDb-shaped configs
(configs[2], configs[3]) on one GPU. Prints one JSON line per point.
Usage: python tools/sweep.py [mnist|fmnist|imdb|all] [q]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_04861_b200 as T  # noqa: E402
from paper_2009_04861_b200 import synth  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"


def run(kind, clauses_list, q, qt, T_, s, epochs=2):
    d = synth.make(kind, q, qt, {"mnist": 2009, "fmnist": 2352, "imdb": 10000}[kind])
    pool = T.ExamplePool(d.features, d.train_x, d.train_y, d.classes)
    test = T.ExamplePool(d.features, d.test_x, d.test_y, d.classes)
    for n in clauses_list:
        tm = T.MultiClassTM(T.TMConfig(clauses=n, margin=T_, specificity=s, seed=42), d.features, d.classes)
        pool.reset_tallies()
        rows = []
        for e in range(epochs):
            t0 = time.perf_counter()
            rep = T.train_epoch_parallel(tm, pool, 1, e)
            wall = time.perf_counter() - t0
            rows.append({"epoch": e, "kernel_ms": rep.device_seconds * 1e3, "wall_ms": wall * 1e3,
                         "events": rep.total_feedback_events(), "type1": sum(rep.type_i_events)})
        acc = T.evaluate_accuracy(tm, test) if qt else None
        m, o = d.classes, d.features
        print(json.dumps({"config": kind, "clauses_per_class": n, "q": q, "T": T_, "s": s, "epochs": rows,
                          "test_accuracy": acc,
                          "clause_literal_evals_per_s_e0": m * n * q * 2 * o / (rows[0]["kernel_ms"] * 1e-3),
                          "examples_per_s_e0": q / (rows[0]["kernel_ms"] * 1e-3)}), flush=True)


q = int(sys.argv[2]) if len(sys.argv) > 2 else 60000


def warm_up():
    """One throwaway epoch so module loading and clock ramp-up stay out of the
    first sweep point."""
    d = synth.make("mnist", 2000, 0, 1)
    tm = T.MultiClassTM(T.TMConfig(clauses=100, margin=50, specificity=10.0, seed=1), 784, 10)
    pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
    T.train_epoch_parallel(tm, pool, 1, 0)


warm_up()
if what in ("mnist", "all"):
    run("mnist", [20, 100, 200, 500, 1000, 2000, 5000, 7000, 10000], q, 10000, 50, 10.0)
if what in ("fmnist", "all"):
    run("fmnist", [8000], q, 10000, 100, 15.0)
if what in ("imdb", "all"):
    run("imdb", [10000], 25000, 25000, 100, 15.0)
