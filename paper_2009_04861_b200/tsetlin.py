"""Python view of the reference's C++ API (namespace ``tsetlin``) over the
B200 C ABI. Names, argument meaning and error classes follow
/root/reference/proj/include/tsetlin/{core,pool,trainer,rng}.hpp so tests
read like the reference's own; every call runs on the GPU through
libtmgpu.so (see _capi.py). There is no host compute path.

Error mapping: std::invalid_argument -> ValueError, std::out_of_range ->
IndexError, runtime/CUDA failures -> TMError.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import check, lib

MODE_ASYNC = _capi.MODE_ASYNC
MODE_SYNC_MIRROR = _capi.MODE_SYNC_MIRROR
MODE_AUTO = _capi.MODE_AUTO
TRAIN, PREDICT = _capi.EVAL_TRAIN, _capi.EVAL_PREDICT  # EvalMode (core.hpp:33-35)


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def literal_words(feature_count: int) -> int:
    """core.hpp:73-75."""
    return (2 * feature_count + 63) // 64


@dataclass
class TMConfig:
    """TMConfig (core.hpp:85-97)."""
    clauses: int = 100
    margin: int = 15
    specificity: float = 3.0
    state_depth: int = 128
    boost_true_positive: bool = False
    epochs: int = 100
    workers: int = 0
    seed: int = 42

    def _c(self) -> _capi.Config:
        return _capi.Config(self.clauses, self.margin, float(self.specificity), self.state_depth,
                            int(bool(self.boost_true_positive)), self.epochs, self.workers,
                            self.seed & (2**64 - 1))

    def validate(self):
        """core.cpp:48-74 — raises ValueError (std::invalid_argument)."""
        c = self._c()
        check(lib().tmg_config_validate(C.byref(c)))

    @staticmethod
    def state_depth_for_bits(bits: int) -> int:
        """``b`` state bits <-> N = 2^(b-1) (8 bits -> the default N=128)."""
        return 1 << (bits - 1)


class Rng:
    """Seedable xoshiro256++ stream (rng.hpp:33-87); state lives on the host
    and is handed to the GPU by update_clause."""

    def __init__(self, seed: int, stream: int = 0):
        self.state = np.zeros(4, np.uint64)
        lib().tmg_rng_state_init(seed & (2**64 - 1), stream & (2**64 - 1), _ptr(self.state))

    def next(self) -> int:
        return int(lib().tmg_rng_state_next(_ptr(self.state)))

    def uniform(self) -> float:
        return (self.next() >> 11) * 2.0**-53


def epoch_order(seed: int, epoch: int, q: int) -> np.ndarray:
    out = np.empty(q, np.int32)
    check(lib().tmg_epoch_order(seed & (2**64 - 1), epoch, q, _ptr(out)))
    return out


class ExamplePool:
    """ExamplePool (pool.hpp:30-78): immutable packed examples + q x m tallies,
    resident on one GPU."""

    def __init__(self, feature_count: int, bits, labels, num_classes: int, device: int = 0):
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        labels = np.ascontiguousarray(labels, dtype=np.int32).reshape(-1)
        q = labels.shape[0]
        if bits.size != q * feature_count:
            if feature_count >= 1 and num_classes >= 1 and q > 0:
                raise ValueError("bit matrix size does not match labels")  # pool.cpp:38-41
        self._h = C.c_void_p()
        check(lib().tmg_pool_create(device, feature_count, _ptr(bits) if bits.size else None,
                                    _ptr(labels) if q else None, q, num_classes, C.byref(self._h)))
        self._o, self._m, self._q, self.device = feature_count, num_classes, q, device
        self._labels = labels.copy()

    @classmethod
    def from_device(cls, feature_count: int, d_bits_ptr: int, d_labels_ptr: int, q: int,
                    num_classes: int, device: int = 0, labels_host=None) -> "ExamplePool":
        self = cls.__new__(cls)
        self._h = C.c_void_p()
        check(lib().tmg_pool_create_device(device, feature_count, d_bits_ptr, d_labels_ptr, q,
                                           num_classes, C.byref(self._h)))
        self._o, self._m, self._q, self.device = feature_count, num_classes, q, device
        self._labels = None if labels_host is None else np.asarray(labels_host, np.int32)
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().tmg_pool_destroy(h)
            except Exception:  # interpreter teardown: the process frees the device anyway
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def size(self) -> int:
        return self._q

    def feature_count(self) -> int:
        return self._o

    def num_classes(self) -> int:
        return self._m

    def words_per_example(self) -> int:
        return literal_words(self._o)

    def all_literals(self) -> np.ndarray:
        out = np.zeros((self._q, literal_words(self._o)), np.uint64)
        check(lib().tmg_pool_get_literals(self._h, _ptr(out)))
        return out

    def literals(self, i: int) -> np.ndarray:
        return self.all_literals()[i]

    def label(self, i: int) -> int:
        return int(self._labels[i])

    def tallies(self) -> np.ndarray:
        out = np.zeros((self._q, self._m), np.int32)
        check(lib().tmg_pool_get_tallies(self._h, _ptr(out)))
        return out

    def tally(self, i: int, c: int) -> int:
        return int(self.tallies()[i, c])

    def set_tallies(self, values: np.ndarray):
        v = np.ascontiguousarray(values, np.int32).reshape(self._q, self._m)
        check(lib().tmg_pool_set_tallies(self._h, _ptr(v)))

    def set_tally(self, i: int, c: int, value: int):
        t = self.tallies()
        t[i, c] = value
        self.set_tallies(t)

    def reset_tallies(self):
        check(lib().tmg_pool_reset_tallies(self._h))

    def tally_device_ptr(self) -> int:
        p = C.c_void_p()
        check(lib().tmg_pool_tally_device_ptr(self._h, C.byref(p)))
        return p.value

    def delta_device_ptr(self) -> int:
        p = C.c_void_p()
        check(lib().tmg_pool_delta_device_ptr(self._h, C.byref(p)))
        return p.value


class ClassBank:
    """Reference ClassBank accessors (core.hpp:110-204) over one bank of a
    device-resident machine."""

    def __init__(self, tm: "MultiClassTM", c: int):
        self._tm, self._c = tm, c

    def feature_count(self) -> int:
        return self._tm.feature_count()

    def literal_count(self) -> int:
        return 2 * self._tm.feature_count()

    def clause_count(self) -> int:
        return self._tm.clause_end - self._tm.clause_begin

    def state_depth(self) -> int:
        return self._tm.config.state_depth

    def words_per_clause(self) -> int:
        return literal_words(self._tm.feature_count())

    def positive(self, j: int) -> bool:
        return j % 2 == 0

    def counters(self) -> np.ndarray:
        out = np.zeros((self.clause_count(), self.literal_count()), np.uint16)
        check(lib().tmg_get_counters(self._tm.handle, self._c, _ptr(out)))
        return out

    def set_counters(self, values: np.ndarray):
        v = np.ascontiguousarray(values, np.uint16).reshape(self.clause_count(), self.literal_count())
        check(lib().tmg_set_counters(self._tm.handle, self._c, _ptr(v)))

    def counter(self, j: int, k: int) -> int:
        return int(self.counters()[j - self._tm.clause_begin, k])

    def set_counter(self, j: int, k: int, value: int):
        cs = self.counters()
        cs[j - self._tm.clause_begin, k] = value
        self.set_counters(cs)

    def include_masks(self) -> np.ndarray:
        out = np.zeros((self.clause_count(), self.words_per_clause()), np.uint64)
        check(lib().tmg_get_include_masks(self._tm.handle, self._c, _ptr(out)))
        return out

    def include_mask(self, j: int) -> np.ndarray:
        return self.include_masks()[j - self._tm.clause_begin]

    def include_counts(self) -> np.ndarray:
        out = np.zeros(self.clause_count(), np.int32)
        check(lib().tmg_get_include_counts(self._tm.handle, self._c, _ptr(out)))
        return out

    def include_count(self, j: int) -> int:
        return int(self.include_counts()[j - self._tm.clause_begin])

    def bound_examples(self) -> int:
        q = C.c_int64()
        check(lib().tmg_bank_bound_examples(self._tm.handle, self._c, C.byref(q)))
        return q.value

    def bind_examples(self, q: int):
        """ClassBank::bind_examples (core.cpp:117-126): this bank only."""
        check(lib().tmg_bind_bank(self._tm.handle, self._c, q))

    def prev_outputs(self) -> np.ndarray:
        q = self.bound_examples()
        out = np.zeros((self.clause_count(), (q + 63) // 64), np.uint64)
        check(lib().tmg_get_prev_outputs(self._tm.handle, self._c, _ptr(out)))
        return out

    def set_prev_outputs(self, values: np.ndarray):
        q = self.bound_examples()
        v = np.ascontiguousarray(values, np.uint64).reshape(self.clause_count(), (q + 63) // 64)
        check(lib().tmg_set_prev_outputs(self._tm.handle, self._c, _ptr(v)))

    def prev_output(self, j: int, i: int) -> bool:
        w = self.prev_outputs()[j - self._tm.clause_begin, i >> 6]
        return bool((int(w) >> (i & 63)) & 1)


class MultiClassTM:
    """MultiClassTM (trainer.hpp:45-54): config + m banks, resident on one GPU.
    ``clause_range`` selects an even-aligned clause shard for multi-GPU."""

    def __init__(self, cfg: TMConfig, feature_count: int, num_classes: int, device: int = 0,
                 clause_range: Optional[Sequence[int]] = None, devices: Optional[Sequence[int]] = None):
        self.config = cfg
        c = cfg._c()
        self._h = C.c_void_p()
        if devices is not None:  # clause shards over several GPUs (repeats: several shards on one GPU)
            devs = (C.c_int32 * len(devices))(*[int(v) for v in devices])
            check(lib().tmg_machine_create_devices(C.byref(c), feature_count, num_classes, devs, len(devices),
                                                   C.byref(self._h)))
            self.clause_begin, self.clause_end = 0, cfg.clauses
            device = int(devices[0])
        elif clause_range is None:
            check(lib().tmg_machine_create(C.byref(c), feature_count, num_classes, device,
                                           C.byref(self._h)))
            self.clause_begin, self.clause_end = 0, cfg.clauses
        else:
            jb, je = int(clause_range[0]), int(clause_range[1])
            check(lib().tmg_machine_create_shard(C.byref(c), feature_count, num_classes, device, jb,
                                                 je, C.byref(self._h)))
            self.clause_begin, self.clause_end = jb, je
        self._o, self._m, self.device = feature_count, num_classes, device
        self.banks = [ClassBank(self, k) for k in range(num_classes)]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().tmg_machine_destroy(h)
            except Exception:  # interpreter teardown: the process frees the device anyway
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def feature_count(self) -> int:
        return self._o

    def num_banks(self) -> int:
        return self._m

    def info(self) -> _capi.MachineInfo:
        inf = _capi.MachineInfo()
        check(lib().tmg_machine_info_get(self._h, C.byref(inf)))
        return inf

    def reset(self):
        check(lib().tmg_machine_reset(self._h))

    def bind_examples(self, q: int):
        check(lib().tmg_bind_examples(self._h, q))

    def set_windows(self, windows: int):
        """Tally-exchange windows per epoch of a sharded machine (default 16)."""
        check(lib().tmg_machine_set_windows(self._h, windows))

    def exchange_info(self):
        """(shards or ranks, whether the exchange runs over NCCL)."""
        n, nccl = C.c_int32(), C.c_int32()
        check(lib().tmg_machine_exchange_info(self._h, C.byref(n), C.byref(nccl)))
        return n.value, bool(nccl.value)

    def attach_comm(self, comm: Optional["Comm"]):
        check(lib().tmg_machine_attach_comm(self._h, comm.handle if comm is not None else None))


class Comm:
    """One rank's NCCL communicator for a multi-process clause-sharded
    machine (tmg_comm_create): rank 0 calls unique_id(), the caller sends the
    128 bytes to every rank (e.g. torch.distributed.broadcast_object_list)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        check(lib().tmg_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        self._h = C.c_void_p()
        check(lib().tmg_comm_create(buf, nranks, rank, device, C.byref(self._h)))

    @classmethod
    def ipc(cls, nranks: int, rank: int, device: int, capacity: int, allgather) -> "Comm":
        """The NCCL-free communicator over CUDA IPC (one node): `capacity` =
        the largest q x m of the machine's pools; `allgather(bytes) -> list of
        bytes` in rank order (e.g. torch.distributed.all_gather_object)."""
        self = cls.__new__(cls)
        self._h = C.c_void_p()
        check(lib().tmg_comm_create_ipc(nranks, rank, device, capacity, C.byref(self._h)))
        h = (C.c_ubyte * 192)()
        check(lib().tmg_comm_ipc_handle(self._h, h))
        handles = allgather(bytes(h))
        buf = (C.c_ubyte * (192 * nranks)).from_buffer_copy(b"".join(handles))
        check(lib().tmg_comm_ipc_connect(self._h, buf))
        return self

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().tmg_comm_destroy(h)
            except Exception:
                pass
            self._h = None


def nccl_available():
    why = C.create_string_buffer(256)
    ok = lib().tmg_nccl_available(why, 256)
    return bool(ok), why.value.decode()


@dataclass
class EpochReport:
    """EpochReport (trainer.hpp:31-43)."""
    epoch: int = 0
    seconds: float = 0.0
    device_seconds: float = 0.0
    feedback_events: List[int] = field(default_factory=list)
    train_metric: Optional[float] = None
    test_metric: Optional[float] = None

    def total_feedback_events(self) -> int:
        return int(sum(self.feedback_events))


def train_epoch_parallel(tm: MultiClassTM, pool: ExamplePool, workers: int, epoch: int,
                         mode: int = MODE_AUTO) -> EpochReport:
    """train_epoch_parallel (trainer.cpp:181-242) on the GPU.

    mode=MODE_ASYNC runs Algorithm 1 over all clauses concurrently;
    mode=MODE_SYNC_MIRROR replays the reference's W-worker schedule with its
    xoshiro streams (bit-exact for workers=1); MODE_AUTO (the default, as in
    the C++ facade) is MODE_ASYNC unless workers == 1 and the environment sets
    TSETLIN_DETERMINISTIC=1."""
    ev = np.zeros(tm.num_banks(), np.uint64)
    ev1 = np.zeros(tm.num_banks(), np.uint64)
    rep = _capi.EpochReportC(0, 0.0, 0.0, ev.ctypes.data_as(C.POINTER(C.c_uint64)),
                             ev1.ctypes.data_as(C.POINTER(C.c_uint64)))
    check(lib().tmg_train_epoch(tm.handle, pool.handle, mode, workers, epoch, C.byref(rep)))
    r = EpochReport(rep.epoch, rep.seconds, rep.device_seconds, [int(v) for v in ev])
    r.type_i_events = [int(v) for v in ev1]
    return r


def train_epoch_sequential(tm: MultiClassTM, pool: ExamplePool, epoch: int) -> EpochReport:
    """train_epoch_sequential (trainer.cpp:138-179), replayed bit-exactly on the GPU."""
    ev = np.zeros(tm.num_banks(), np.uint64)
    secs = C.c_double(0)
    check(lib().tmg_train_epoch_sequential(tm.handle, pool.handle, epoch, C.byref(secs), _ptr(ev)))
    return EpochReport(epoch, secs.value, secs.value, [int(v) for v in ev])


def update_clause(bank: ClassBank, j: int, pool: ExamplePool, class_idx: int, order, offset: int,
                  batch: int, margin: int, s: float, boost_true_positive: bool, rng: Rng) -> int:
    """update_clause (trainer.cpp:102-136) with the reference stream `rng`."""
    if bank._c != class_idx:
        raise ValueError("bank does not belong to class_idx")
    o = None if order is None or len(order) == 0 else np.ascontiguousarray(order, np.int32)
    ev = C.c_uint64(0)
    check(lib().tmg_update_clause(bank._tm.handle, pool.handle, class_idx, j,
                                  _ptr(o) if o is not None else None, 0 if o is None else len(o),
                                  offset, batch, margin, float(s), int(bool(boost_true_positive)),
                                  _ptr(rng.state), C.byref(ev)))
    return int(ev.value)


def refresh_tallies(pool: ExamplePool, tm: MultiClassTM):
    """refresh_tallies (pool.cpp:108-124); banks are the machine's."""
    check(lib().tmg_refresh_tallies(tm.handle, pool.handle))


def class_sums(tm: MultiClassTM, pool: ExamplePool, mode: int = PREDICT) -> np.ndarray:
    """export_vote_sums (trainer.cpp:262-270) for every example of a pool."""
    out = np.zeros((pool.size(), tm.num_banks()), np.int32)
    check(lib().tmg_class_sums(tm.handle, pool.handle, mode, _ptr(out)))
    return out


def _lits2d(tm: MultiClassTM, literals) -> np.ndarray:
    lits = np.ascontiguousarray(literals, np.uint64)
    if lits.ndim == 1:
        lits = lits[None, :]
    if lits.shape[1] != literal_words(tm.feature_count()):
        raise ValueError("literal row width does not match the machine")
    return lits


def export_vote_sums(tm: MultiClassTM, literals) -> np.ndarray:
    """export_vote_sums (trainer.cpp:262-270). 1-D row -> m sums; 2-D -> q x m."""
    lits = _lits2d(tm, literals)
    out = np.zeros((lits.shape[0], tm.num_banks()), np.int32)
    check(lib().tmg_class_sums_literals(tm.handle, _ptr(lits), lits.shape[0], PREDICT, _ptr(out)))
    return out[0] if np.asarray(literals).ndim == 1 else out


def vote_sum(bank: ClassBank, literals, mode: int) -> int:
    """vote_sum (pool.cpp:82-91) of one bank on one literal row."""
    lits = _lits2d(bank._tm, literals)
    out = np.zeros((1, bank._tm.num_banks()), np.int32)
    check(lib().tmg_class_sums_literals(bank._tm.handle, _ptr(lits[:1]), 1, mode, _ptr(out)))
    return int(out[0, bank._c])


def classify(tm: MultiClassTM, literals) -> int:
    """classify (trainer.cpp:244-260)."""
    lits = _lits2d(tm, literals)
    out = np.zeros(1, np.int32)
    check(lib().tmg_predict_literals(tm.handle, _ptr(lits[:1]), 1, _ptr(out)))
    return int(out[0])


def predict_all(tm: MultiClassTM, pool: ExamplePool) -> np.ndarray:
    """predict_all (trainer.cpp:272-279)."""
    out = np.zeros(pool.size(), np.int32)
    check(lib().tmg_predict(tm.handle, pool.handle, _ptr(out)))
    return out


def predict_literals(tm: MultiClassTM, literals) -> np.ndarray:
    lits = _lits2d(tm, literals)
    out = np.zeros(lits.shape[0], np.int32)
    check(lib().tmg_predict_literals(tm.handle, _ptr(lits), lits.shape[0], _ptr(out)))
    return out


def evaluate_accuracy(tm: MultiClassTM, pool: ExamplePool, labels=None) -> float:
    """evaluate_accuracy (trainer.cpp:281-287)."""
    pred = predict_all(tm, pool)
    y = pool._labels if labels is None else np.asarray(labels, np.int32)
    return float(np.mean(pred == y))


def device_count() -> int:
    n = C.c_int32(0)
    check(lib().tmg_device_count(C.byref(n)))
    return int(n.value)


def _feedback(bank: ClassBank, j: int, literals, kind: int, s: float, boost: bool, rng: Optional[Rng]):
    lits = _lits2d(bank._tm, literals)[:1].copy()
    state = rng.state if rng is not None else np.zeros(4, np.uint64)
    check(lib().tmg_feedback(bank._tm.handle, bank._c, j, _ptr(lits), kind, float(s), int(bool(boost)),
                             -1, _ptr(state)))


def feedback_rates(bank: ClassBank, j: int, literals, clause_output: int, trials: int):
    """Per-literal +1/-1 transition counts of the async Type I path over
    `trials` independent applications (statistical conformance probe)."""
    lits = _lits2d(bank._tm, literals)[:1].copy()
    L = bank.literal_count()
    inc, dec = np.zeros(L, np.uint64), np.zeros(L, np.uint64)
    check(lib().tmg_debug_feedback_rates(bank._tm.handle, bank._c, j, _ptr(lits), int(clause_output), trials,
                                         _ptr(inc), _ptr(dec)))
    return inc, dec


def type_i_async(bank: ClassBank, j: int, literals, clause_output: int, example: int, epoch: int):
    """One asynchronous Type I feedback on clause j (the epoch kernel's Philox
    sampler, counters (clause, example), key of `epoch`), applied in place."""
    lits = _lits2d(bank._tm, literals)[:1].copy()
    check(lib().tmg_debug_type_i_async(bank._tm.handle, bank._c, j, _ptr(lits), int(clause_output),
                                       int(example) & 0xFFFFFFFF, int(epoch)))


def alias8_table(threshold: int) -> np.ndarray:
    """The engine's 256-entry alias table for clause-output-0 Type I draws at
    feed-back probability threshold / 2^32 (host computation)."""
    out = np.zeros(256, np.uint32)
    check(lib().tmg_alias8_table(int(threshold) & 0xFFFFFFFF, _ptr(out)))
    return out


def evaluate_clause(bank: ClassBank, j: int, literals, mode: int) -> int:
    """evaluate_clause (core.hpp:208-219) on the GPU."""
    lits = _lits2d(bank._tm, literals)[:1].copy()
    out = C.c_int32(0)
    check(lib().tmg_evaluate_clause(bank._tm.handle, bank._c, j, _ptr(lits), mode, C.byref(out)))
    return int(out.value)


def type_i_feedback(bank: ClassBank, j: int, literals, s: float, boost_true_positive: bool, rng: Rng):
    """type_i_feedback (feedback.cpp:87-93): one uniform per literal from rng."""
    _feedback(bank, j, literals, 1, s, boost_true_positive, rng)


def type_ii_feedback(bank: ClassBank, j: int, literals):
    """type_ii_feedback (feedback.cpp:95-99)."""
    _feedback(bank, j, literals, 2, 1.0, False, None)


def kernel_launches() -> int:
    """Kernels launched by libtmgpu.so in this process so far."""
    return int(lib().tmg_kernel_launches())


def machine_stream(tm: MultiClassTM) -> int:
    """cudaStream_t (as an int) the machine's work is enqueued on."""
    p = C.c_void_p()
    check(lib().tmg_machine_stream(tm.handle, C.byref(p)))
    return p.value or 0


def int_peak(device: int = 0):
    """Measured integer-pipe peaks (thread-ops/s): (LOP3 only, LOP3+IMAD)."""
    a, b = C.c_double(0), C.c_double(0)
    check(lib().tmg_bench_int_peak(device, C.byref(a), C.byref(b)))
    return a.value, b.value


# ------------------------------------------------------------ regression ---
class RegressionHead:
    """RegressionHead (regression.hpp:26-35): one all-positive bank whose
    clipped clause count decodes linearly into [y_min, y_max]."""

    def __init__(self, cfg: TMConfig, feature_count: int, y_min: float, y_max: float, device: int = 0):
        cfg.validate()
        if not (y_max > y_min):
            raise ValueError("target range must satisfy y_max > y_min")
        self.config, self.y_min, self.y_max, self.device = cfg, float(y_min), float(y_max), device
        c = cfg._c()
        self._h = C.c_void_p()
        check(lib().tmg_machine_create_regress(C.byref(c), feature_count, device, C.byref(self._h)))
        self._o = feature_count
        self.clause_begin, self.clause_end = 0, cfg.clauses
        self.bank = ClassBank(self, 0)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().tmg_machine_destroy(h)
            except Exception:  # interpreter teardown: the process frees the device anyway
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def feature_count(self) -> int:
        return self._o

    def num_banks(self) -> int:
        return 1

    def info(self) -> _capi.MachineInfo:
        inf = _capi.MachineInfo()
        check(lib().tmg_machine_info_get(self._h, C.byref(inf)))
        return inf


def scaled_target(head: RegressionHead, y: float) -> int:
    """regression.cpp:82-89 (round half away from zero, like std::lround)."""
    if y < head.y_min or y > head.y_max:
        raise ValueError("target outside [y_min, y_max]")
    v = (y - head.y_min) * head.config.margin / (head.y_max - head.y_min)
    return int(np.floor(v + 0.5)) if v >= 0 else -int(np.floor(-v + 0.5))


def regress_pool(head: RegressionHead, bits, targets, device: int = 0) -> ExamplePool:
    """ExamplePool of scaled targets (one tally class) for a regression head."""
    scaled = np.array([scaled_target(head, float(y)) for y in np.asarray(targets).reshape(-1)], np.int32)
    return ExamplePool(head.feature_count(), bits, scaled, 1, device=device)


def predict_scaled_all(head: RegressionHead, pool: ExamplePool) -> np.ndarray:
    """predict_scaled (regression.cpp:86-93) for every pool example."""
    out = np.zeros(pool.size(), np.int32)
    check(lib().tmg_regress_predict(head.handle, pool.handle, _ptr(out)))
    return out


def predict_scaled(head: RegressionHead, literals) -> int:
    lits = _lits2d(head, literals)[:1].copy()
    out = np.zeros(1, np.int32)
    check(lib().tmg_regress_predict_literals(head.handle, _ptr(lits), 1, _ptr(out)))
    return int(out[0])


def predict_regress(head: RegressionHead, literals) -> float:
    """regression.cpp:95-99."""
    v = predict_scaled(head, literals)
    return head.y_min + v * (head.y_max - head.y_min) / head.config.margin


def update_regress(head: RegressionHead, literals, y_target: float, rng: Rng) -> int:
    """update_regress (regression.cpp:101-123) with the reference stream."""
    t = scaled_target(head, y_target)
    lits = _lits2d(head, literals)[:1].copy()
    ev = C.c_uint64(0)
    check(lib().tmg_update_regress(head.handle, _ptr(lits), t, _ptr(rng.state), C.byref(ev)))
    return int(ev.value)


def train_epoch_regress_sequential(head: RegressionHead, pool: ExamplePool, epoch: int) -> EpochReport:
    ev = np.zeros(1, np.uint64)
    secs = C.c_double(0)
    check(lib().tmg_train_epoch_regress_sequential(head.handle, pool.handle, epoch, C.byref(secs), _ptr(ev)))
    return EpochReport(epoch, secs.value, secs.value, [int(ev[0])])


def train_epoch_regress_parallel(head: RegressionHead, pool: ExamplePool, workers: int, epoch: int,
                                 mode: int = MODE_AUTO) -> EpochReport:
    ev = np.zeros(1, np.uint64)
    ev1 = np.zeros(1, np.uint64)
    rep = _capi.EpochReportC(0, 0.0, 0.0, ev.ctypes.data_as(C.POINTER(C.c_uint64)),
                             ev1.ctypes.data_as(C.POINTER(C.c_uint64)))
    check(lib().tmg_train_epoch_regress(head.handle, pool.handle, mode, workers, epoch, C.byref(rep)))
    r = EpochReport(rep.epoch, rep.seconds, rep.device_seconds, [int(ev[0])])
    r.type_i_events = [int(ev1[0])]
    return r


def evaluate_scaled_mae(head: RegressionHead, pool: ExamplePool, targets=None) -> float:
    """regression.cpp:229-236 (pool labels are the scaled targets)."""
    pred = predict_scaled_all(head, pool)
    t = pool._labels if targets is None else np.asarray(targets, np.int32)
    return float(np.mean(np.abs(pred.astype(np.int64) - t)))
