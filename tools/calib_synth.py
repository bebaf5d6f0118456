#!/usr/bin/env python3
"""Calibrates the FMNIST- and IMDb-shaped generators (csrc/synth.c) to be
non-saturating: GPU async training, n clauses/class, 2 epochs, test accuracy
per parameter set. One JSON line per setting."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_04861_b200 as T  # noqa: E402
from paper_2009_04861_b200._capi import lib  # noqa: E402


def fmnist(r_class, r_sub, amp, mix, q, qt):
    tx, ty = np.zeros((q, 2352), np.uint8), np.zeros(q, np.int32)
    vx, vy = np.zeros((qt, 2352), np.uint8), np.zeros(qt, np.int32)
    assert lib().tmg_synth_fmnist(2352, 784, 10, r_class, r_sub, amp, mix, q, qt, tx.ctypes.data,
                                  ty.ctypes.data, vx.ctypes.data, vy.ctypes.data) == 0
    return tx, ty, vx, vy


def imdb(p_sent, cross, q, qt):
    tx, ty = np.zeros((q, 10000), np.uint8), np.zeros(q, np.int32)
    vx, vy = np.zeros((qt, 10000), np.uint8), np.zeros(qt, np.int32)
    assert lib().tmg_synth_imdb(10000, 10000, 250, p_sent, cross, q, qt, tx.ctypes.data, ty.ctypes.data,
                                vx.ctypes.data, vy.ctypes.data) == 0
    return tx, ty, vx, vy


def trial(data, m, n, T_, s, epochs=2):
    tx, ty, vx, vy = data
    o = tx.shape[1]
    tm = T.MultiClassTM(T.TMConfig(clauses=n, margin=T_, specificity=s, seed=42), o, m)
    pool, test = T.ExamplePool(o, tx, ty, m), T.ExamplePool(o, vx, vy, m)
    accs = []
    for e in range(epochs):
        T.train_epoch_parallel(tm, pool, 1, e)
        accs.append(T.evaluate_accuracy(tm, test))
    return accs


for rc, rs, amp, mix in [(0.10, 0.15, 60, 0.8), (0.10, 0.15, 60, 0.9), (0.10, 0.15, 90, 0.95),
                         (0.05, 0.15, 60, 0.9)]:
    print(json.dumps({"fmnist": [rc, rs, amp, mix],
                      "acc": trial(fmnist(rc, rs, amp, mix, 10000, 2000), 10, 2000, 100, 15.0)}), flush=True)
for ps, cr in [(0.10, 0.3), (0.15, 0.3), (0.08, 0.2), (0.2, 0.4)]:
    print(json.dumps({"imdb": [ps, cr], "acc": trial(imdb(ps, cr, 5000, 2000), 2, 2000, 100, 15.0)}), flush=True)
