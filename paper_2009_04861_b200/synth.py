"""Synthetic datasets for the BASELINE.json configs (csrc/synth.c via the C
ABI). Identical bytes to what oracle/_ref/ref_driver trains on."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._capi import lib


@dataclass
class Split:
    features: int
    classes: int
    train_x: np.ndarray
    train_y: np.ndarray
    test_x: np.ndarray
    test_y: np.ndarray


def _alloc(q, o):
    return np.zeros((q, o), np.uint8), np.zeros(q, np.int32)


def make(kind: str, q: int, qt: int, seed: int, noise: float = 0.0) -> Split:
    """The canonical presets of csrc/synth.c (tmg_synth_preset), shared with
    oracle/ref_driver.cpp make_data()."""
    shapes = {"xor": (0, 12, 2), "mnist": (1, 784, 10), "fmnist": (2, 2352, 10), "imdb": (3, 10000, 2)}
    if kind not in shapes:
        raise ValueError(f"unknown dataset {kind}")
    k, o, m = shapes[kind]
    tx, ty = _alloc(q, o)
    vx, vy = _alloc(qt, o)
    assert lib().tmg_synth_preset(k, seed, noise, q, qt, tx.ctypes.data, ty.ctypes.data, vx.ctypes.data,
                                  vy.ctypes.data) == 0
    return Split(o, m, tx, ty, vx, vy)
