"""ctypes wrapper over oracle/_build/liboracle.so (the C restatement).

TEST INFRASTRUCTURE ONLY — the checker. Imported by tests/, by
__graft_entry__.smoke() and by bench.py's cpu_baseline leg; never by the
product package. Parity of the restatement is pinned against the compiled
reference's golden dumps (tests/test_oracle_golden.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
REF_DRIVER = os.path.join(HERE, "_ref", "ref_driver")


class _Rng(C.Structure):
    _fields_ = [("s", C.c_uint64 * 4)]


class _Machine(C.Structure):
    _fields_ = [("o", C.c_int32), ("L", C.c_int32), ("m", C.c_int32), ("n", C.c_int32),
                ("N", C.c_int32), ("W64", C.c_int32), ("q_bound", C.c_int32),
                ("out_words", C.c_int32), ("counters", C.c_void_p), ("masks", C.c_void_p),
                ("counts", C.c_void_p), ("prev", C.c_void_p)]


class _Pool(C.Structure):
    _fields_ = [("o", C.c_int32), ("m", C.c_int32), ("W64", C.c_int32), ("q", C.c_int64),
                ("lits", C.c_void_p), ("labels", C.c_void_p), ("tallies", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.orc_rng_init.argtypes = [C.POINTER(_Rng), C.c_uint64, C.c_uint64]
        L.orc_rng_next.argtypes = [C.POINTER(_Rng)]
        L.orc_rng_next.restype = C.c_uint64
        L.orc_rng_uniform.argtypes = [C.POINTER(_Rng)]
        L.orc_rng_uniform.restype = C.c_double
        L.orc_rng_below.argtypes = [C.POINTER(_Rng), C.c_uint32]
        L.orc_rng_below.restype = C.c_uint32
        L.orc_shuffled_indices.argtypes = [C.c_int32, C.POINTER(_Rng), P]
        L.orc_mix_stream.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_mix_stream.restype = C.c_uint64
        L.orc_clause_offset.argtypes = [C.c_uint64, C.c_int64]
        L.orc_clause_offset.restype = C.c_uint64
        L.orc_pack_literals.argtypes = [C.c_int32, P, P]
        L.orc_clause_update_probability.argtypes = [C.c_int32, C.c_int32, C.c_int32]
        L.orc_clause_update_probability.restype = C.c_double
        L.orc_rebuild_masks.argtypes = [C.POINTER(_Machine)]
        L.orc_evaluate_clause.argtypes = [C.POINTER(_Machine), C.c_int, C.c_int, P, C.c_int]
        L.orc_type_i.argtypes = [C.POINTER(_Machine), C.c_int, C.c_int, P, C.c_int, C.c_double,
                                 C.c_int, C.POINTER(_Rng)]
        L.orc_type_ii.argtypes = [C.POINTER(_Machine), C.c_int, C.c_int, P, C.c_int]
        L.orc_bind.argtypes = [C.POINTER(_Machine), C.c_int32]
        L.orc_update_clause.argtypes = [C.POINTER(_Machine), C.POINTER(_Pool), C.c_int, C.c_int, P,
                                        C.c_int64, C.c_int64, C.c_int32, C.c_double, C.c_int,
                                        C.POINTER(_Rng)]
        L.orc_update_clause.restype = C.c_uint64
        L.orc_train_epoch_parallel.argtypes = [C.POINTER(_Machine), C.POINTER(_Pool), C.c_int32,
                                               C.c_double, C.c_int, C.c_uint64, C.c_int32,
                                               C.c_int32, P]
        L.orc_train_epoch_sequential.argtypes = [C.POINTER(_Machine), C.POINTER(_Pool), C.c_int32,
                                                 C.c_double, C.c_int, C.c_uint64, C.c_int32, P]
        L.orc_class_sums.argtypes = [C.POINTER(_Machine), P, C.c_int64, P]
        L.orc_predict.argtypes = [C.POINTER(_Machine), P, C.c_int64, P]
        L.orc_refresh_tallies.argtypes = [C.POINTER(_Machine), C.POINTER(_Pool)]
        L.orc_update_regress.argtypes = [C.POINTER(_Machine), P, C.c_int32, C.c_int32, C.c_double, C.c_int,
                                         C.POINTER(_Rng)]
        L.orc_update_regress.restype = C.c_uint64
        L.orc_train_epoch_regress_sequential.argtypes = [C.POINTER(_Machine), C.POINTER(_Pool), C.c_int32,
                                                         C.c_double, C.c_int, C.c_uint64, C.c_int32]
        L.orc_train_epoch_regress_sequential.restype = C.c_uint64
        L.orc_train_epoch_regress_parallel.argtypes = [C.POINTER(_Machine), C.POINTER(_Pool), C.c_int32,
                                                       C.c_double, C.c_int, C.c_uint64, C.c_int32, C.c_int32]
        L.orc_train_epoch_regress_parallel.restype = C.c_uint64
        L.orc_predict_scaled.argtypes = [C.POINTER(_Machine), P, C.c_int64, C.c_int32, P]
        L.orc_philox4x32.argtypes = [P, C.c_uint32, C.c_uint32, C.c_int, P]
        L.orc_async_key.argtypes = [C.c_uint64, C.c_int32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.orc_async_type_i.argtypes = [P, P, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_int32,
                                       C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int32, C.c_int32, P]
        L.orc_prob_threshold.argtypes = [C.c_double]
        L.orc_prob_threshold.restype = C.c_uint32
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


class Rng:
    """xoshiro256++ stream (reference rng.hpp:33-87)."""

    def __init__(self, seed: int, stream: int = 0, state=None):
        self._r = _Rng()
        if state is not None:
            for k in range(4):
                self._r.s[k] = int(state[k])
        else:
            lib().orc_rng_init(C.byref(self._r), seed & (2**64 - 1), stream & (2**64 - 1))

    @property
    def state(self):
        return [int(self._r.s[k]) for k in range(4)]

    def next(self) -> int:
        return int(lib().orc_rng_next(C.byref(self._r)))

    def uniform(self) -> float:
        return float(lib().orc_rng_uniform(C.byref(self._r)))

    def below(self, bound: int) -> int:
        return int(lib().orc_rng_below(C.byref(self._r), bound))

    def shuffled_indices(self, count: int) -> np.ndarray:
        out = np.empty(count, np.int32)
        lib().orc_shuffled_indices(count, C.byref(self._r), _ptr(out))
        return out


def words64(o: int) -> int:
    return (2 * o + 63) // 64


def pack_literals(bits: np.ndarray) -> np.ndarray:
    """q x o uint8 -> q x ceil(2o/64) uint64 (reference layout)."""
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    if bits.ndim == 1:
        bits = bits[None, :]
    q, o = bits.shape
    out = np.zeros((q, words64(o)), np.uint64)
    for i in range(q):
        lib().orc_pack_literals(o, _ptr(bits[i]), _ptr(out[i]))
    return out


def clause_update_probability(v: int, y: int, margin: int) -> float:
    return float(lib().orc_clause_update_probability(v, y, margin))


def mix_stream(kind, a, b=0):
    return int(lib().orc_mix_stream(kind, a, b))


def clause_offset(g, q):
    return int(lib().orc_clause_offset(g, q))


class Machine:
    """Reference-layout machine state for m banks of n clauses over o features."""

    def __init__(self, o: int, m: int, n: int, N: int = 128, q: int = 0):
        self.o, self.m, self.n, self.N = o, m, n, N
        self.L = 2 * o
        self.W64 = words64(o)
        self.counters = np.full((m, n, self.L), N, np.uint16)
        self.masks = np.zeros((m, n, self.W64), np.uint64)
        self.counts = np.zeros((m, n), np.int32)
        self.prev = np.zeros((m, n, 0), np.uint64)
        self._s = _Machine()
        self.bind(q)

    def bind(self, q: int):
        self.prev = np.zeros((self.m, self.n, (q + 63) // 64), np.uint64)
        self._sync()
        self._s.q_bound = q
        self._s.out_words = (q + 63) // 64

    def _sync(self):
        s = self._s
        s.o, s.L, s.m, s.n, s.N, s.W64 = self.o, self.L, self.m, self.n, self.N, self.W64
        s.out_words = self.prev.shape[2]
        s.counters, s.masks = _ptr(self.counters), _ptr(self.masks)
        s.counts, s.prev = _ptr(self.counts), _ptr(self.prev)
        return C.byref(s)

    def set_counters(self, counters: np.ndarray):
        self.counters[...] = counters
        lib().orc_rebuild_masks(self._sync())

    def evaluate(self, c, j, lits, mode=0):
        lits = np.ascontiguousarray(lits, np.uint64)
        return int(lib().orc_evaluate_clause(self._sync(), c, j, _ptr(lits), mode))

    def type_i(self, c, j, lits, out, s, boost, rng: Rng):
        lits = np.ascontiguousarray(lits, np.uint64)
        lib().orc_type_i(self._sync(), c, j, _ptr(lits), out, s, int(boost), C.byref(rng._r))

    def type_ii(self, c, j, lits, out):
        lits = np.ascontiguousarray(lits, np.uint64)
        lib().orc_type_ii(self._sync(), c, j, _ptr(lits), out)

    def class_sums(self, lits: np.ndarray) -> np.ndarray:
        lits = np.ascontiguousarray(lits, np.uint64)
        out = np.zeros((lits.shape[0], self.m), np.int32)
        lib().orc_class_sums(self._sync(), _ptr(lits), lits.shape[0], _ptr(out))
        return out

    def predict(self, lits: np.ndarray) -> np.ndarray:
        lits = np.ascontiguousarray(lits, np.uint64)
        out = np.zeros(lits.shape[0], np.int32)
        lib().orc_predict(self._sync(), _ptr(lits), lits.shape[0], _ptr(out))
        return out


class Pool:
    def __init__(self, bits: np.ndarray, labels: np.ndarray, m: int):
        self.bits = np.ascontiguousarray(bits, np.uint8)
        self.q, self.o = self.bits.shape
        self.m = m
        self.lits = pack_literals(self.bits)
        self.labels = np.ascontiguousarray(labels, np.int32)
        self.tallies = np.zeros((self.q, m), np.int32)
        self._s = _Pool()

    def _sync(self):
        s = self._s
        s.o, s.m, s.W64, s.q = self.o, self.m, self.lits.shape[1], self.q
        s.lits, s.labels, s.tallies = _ptr(self.lits), _ptr(self.labels), _ptr(self.tallies)
        return C.byref(s)


def update_clause(tm: Machine, pool: Pool, c, j, order, offset, batch, margin, s, boost, rng: Rng):
    if tm._s.q_bound != pool.q:
        tm.bind(pool.q)
    o = None if order is None or len(order) == 0 else np.ascontiguousarray(order, np.int32)
    return int(lib().orc_update_clause(tm._sync(), pool._sync(), c, j, _ptr(o) if o is not None else None,
                                       offset, batch, margin, s, int(boost), C.byref(rng._r)))


def train_epoch_parallel(tm: Machine, pool: Pool, margin, s, boost, seed, workers, epoch):
    if tm._s.q_bound != pool.q:
        tm.bind(pool.q)
    ev = np.zeros(tm.m, np.uint64)
    lib().orc_train_epoch_parallel(tm._sync(), pool._sync(), margin, s, int(boost), seed, workers,
                                   epoch, _ptr(ev))
    return ev


def train_epoch_sequential(tm: Machine, pool: Pool, margin, s, boost, seed, epoch):
    ev = np.zeros(tm.m, np.uint64)
    lib().orc_train_epoch_sequential(tm._sync(), pool._sync(), margin, s, int(boost), seed, epoch,
                                     _ptr(ev))
    return ev


def train_epoch_regress_sequential(tm: Machine, pool: Pool, margin, s, boost, seed, epoch) -> int:
    return int(lib().orc_train_epoch_regress_sequential(tm._sync(), pool._sync(), margin, s, int(boost), seed,
                                                        epoch))


def train_epoch_regress_parallel(tm: Machine, pool: Pool, margin, s, boost, seed, workers, epoch) -> int:
    if tm._s.q_bound != pool.q:
        tm.bind(pool.q)
    return int(lib().orc_train_epoch_regress_parallel(tm._sync(), pool._sync(), margin, s, int(boost), seed,
                                                      workers, epoch))


def update_regress(tm: Machine, lits, t, margin, s, boost, rng: Rng) -> int:
    lits = np.ascontiguousarray(lits, np.uint64)
    return int(lib().orc_update_regress(tm._sync(), _ptr(lits), t, margin, s, int(boost), C.byref(rng._r)))


def predict_scaled(tm: Machine, lits, margin) -> np.ndarray:
    lits = np.ascontiguousarray(lits, np.uint64)
    out = np.zeros(lits.shape[0], np.int32)
    lib().orc_predict_scaled(tm._sync(), _ptr(lits), lits.shape[0], margin, _ptr(out))
    return out


def refresh_tallies(tm: Machine, pool: Pool):
    if tm._s.q_bound != pool.q:
        tm.bind(pool.q)
    lib().orc_refresh_tallies(tm._sync(), pool._sync())


def philox4x32(ctr, key0: int, key1: int, rounds: int = 7) -> np.ndarray:
    """Philox4x32-R block (tm_oracle_async.c), the async engine's generator."""
    c = np.ascontiguousarray(ctr, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32(_ptr(c), key0, key1, rounds, _ptr(out))
    return out


def async_key(seed: int, epoch: int):
    """Philox key (key0, key1) of an async epoch."""
    k0, k1 = C.c_uint32(0), C.c_uint32(0)
    lib().orc_async_key(seed, epoch, C.byref(k0), C.byref(k1))
    return int(k0.value), int(k1.value)


def prob_threshold(p: float) -> int:
    """P(u < p) as a 32-bit fixed-point threshold (the async engine's)."""
    return int(lib().orc_prob_threshold(p))


def async_type_i(counters_row: np.ndarray, lits_row: np.ndarray, o: int, N: int, out: int, s: float,
                 boost: bool, g: int, i: int, seed: int, epoch: int, nw: int, rounds: int = 7,
                 alias8=None) -> np.ndarray:
    """One async-engine Type I feedback on one clause's 2o counters (copy).
    alias8: the engine's 256-entry table for clause output 0 (None: bit-serial)."""
    row = np.ascontiguousarray(counters_row, np.uint16).copy()
    lits = np.ascontiguousarray(lits_row, np.uint64)
    k0, k1 = async_key(seed, epoch)
    tab = None if alias8 is None else np.ascontiguousarray(alias8, np.uint32)
    lib().orc_async_type_i(_ptr(row), _ptr(lits), o, N, int(out), float(s), int(bool(boost)), g, i, k0, k1,
                           nw, rounds, None if tab is None else _ptr(tab))
    return row


def alias8_law(table: np.ndarray) -> np.ndarray:
    """Pattern law (256 probabilities) implied by an alias table as the
    engine samples it: column u & 0xFF, own pattern iff (u|0xFF) < entry."""
    law = np.zeros(256)
    for col in range(256):
        e = int(table[col])
        if (e & 0xFF) == col and (e >> 8) == 0:
            law[col] += 1.0 / 256
            continue
        t = (e >> 8) / 2.0 ** 24
        law[col] += t / 256
        law[e & 0xFF] += (1.0 - t) / 256
    return law
