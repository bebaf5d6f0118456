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
    """Same recipes and seeds as oracle/ref_driver.cpp make_data()."""
    if kind == "xor":
        o, m = 12, 2
        tx, ty = _alloc(q, o)
        vx, vy = _alloc(qt, o)
        assert lib().tmg_synth_xor(seed, q, o, noise, 1, tx.ctypes.data, ty.ctypes.data) == 0
        assert lib().tmg_synth_xor(seed + 1000003, qt, o, noise, 0, vx.ctypes.data, vy.ctypes.data) == 0
    elif kind == "mnist":
        o, m = 784, 10
        tx, ty = _alloc(q, o)
        vx, vy = _alloc(qt, o)
        assert lib().tmg_synth_mnist(seed, 784, 10, 0.10, 0.10, 0.30, q, qt, tx.ctypes.data,
                                     ty.ctypes.data, vx.ctypes.data, vy.ctypes.data) == 0
    elif kind == "fmnist":
        o, m = 2352, 10
        tx, ty = _alloc(q, o)
        vx, vy = _alloc(qt, o)
        assert lib().tmg_synth_fmnist(seed, 784, 10, 0.10, 0.15, 40, q, qt, tx.ctypes.data,
                                      ty.ctypes.data, vx.ctypes.data, vy.ctypes.data) == 0
    elif kind == "imdb":
        o, m = 10000, 2
        tx, ty = _alloc(q, o)
        vx, vy = _alloc(qt, o)
        assert lib().tmg_synth_imdb(seed, 10000, 250, 0.04, 0.5, q, qt, tx.ctypes.data,
                                    ty.ctypes.data, vx.ctypes.data, vy.ctypes.data) == 0
    else:
        raise ValueError(f"unknown dataset {kind}")
    return Split(o, m, tx, ty, vx, vy)
