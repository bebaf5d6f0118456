"""ctypes declarations of the C ABI in include/tmgpu.h (libtmgpu.so).

The library is built in-tree (paper_2009_04861_b200/_lib/libtmgpu.so) by
``__graft_entry__.build()`` / ``make -C paper_2009_04861_b200/csrc``. There is
no CPU fallback: if the library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# TMG_LIB selects another build of the engine (tools/build_variants.sh variants).
LIB_PATH = os.environ.get("TMG_LIB") or os.path.join(HERE, "_lib", "libtmgpu.so")

TMG_OK, TMG_EINVAL, TMG_ERANGE, TMG_ERUNTIME = 0, 1, 2, 3
MODE_ASYNC, MODE_SYNC_MIRROR, MODE_AUTO = 0, 1, 2
EVAL_TRAIN, EVAL_PREDICT = 0, 1


class Config(C.Structure):
    _fields_ = [("clauses", C.c_int32), ("margin", C.c_int32), ("specificity", C.c_double),
                ("state_depth", C.c_int32), ("boost_true_positive", C.c_int32),
                ("epochs", C.c_int32), ("workers", C.c_int32), ("seed", C.c_uint64)]


class EpochReportC(C.Structure):
    _fields_ = [("epoch", C.c_int32), ("seconds", C.c_double), ("device_seconds", C.c_double),
                ("feedback_events", C.POINTER(C.c_uint64)),
                ("type_i_events", C.POINTER(C.c_uint64))]


class MachineInfo(C.Structure):
    _fields_ = [("feature_count", C.c_int32), ("num_classes", C.c_int32), ("clauses", C.c_int32),
                ("state_depth", C.c_int32), ("clause_begin", C.c_int32), ("clause_end", C.c_int32),
                ("planes", C.c_int32), ("words_per_lane", C.c_int32),
                ("bound_examples", C.c_int32), ("device", C.c_int32), ("device_bytes", C.c_uint64)]


P = C.c_void_p
I32, I64, U64, D = C.c_int32, C.c_int64, C.c_uint64, C.c_double
PP = C.POINTER(C.c_void_p)

# name -> (restype, argtypes); every symbol here is declared in include/tmgpu.h.
SIGNATURES = {
    "tmg_abi_version": (C.c_int, []),
    "tmg_last_error": (C.c_char_p, []),
    "tmg_device_count": (C.c_int, [C.POINTER(I32)]),
    "tmg_kernel_launches": (C.c_ulonglong, []),
    "tmg_machine_stream": (C.c_int, [P, PP]),
    "tmg_bench_int_peak": (C.c_int, [I32, C.POINTER(D), C.POINTER(D)]),
    "tmg_debug_xoshiro_jump": (C.c_int, [P, C.c_uint64]),
    "tmg_debug_feedback_rates": (C.c_int, [P, I32, I32, P, I32, C.c_uint32, P, P]),
    "tmg_debug_type_i_async": (C.c_int, [P, I32, I32, P, I32, C.c_uint32, I32]),
    "tmg_debug_counters": (C.c_int, [P, P, I32, I32]),
    "tmg_train_window_async": (C.c_int, [P, P, I32, I64, I64]),
    "tmg_window_delta_snapshot": (C.c_int, [P, P, P]),
    "tmg_window_apply_remote": (C.c_int, [P, P, P, P]),
    "tmg_epoch_events": (C.c_int, [P, P]),
    "tmg_alias8_table": (C.c_int, [C.c_uint32, P]),
    "tmg_config_default": (None, [C.POINTER(Config)]),
    "tmg_config_validate": (C.c_int, [C.POINTER(Config)]),
    "tmg_effective_workers": (I32, [C.POINTER(Config)]),
    "tmg_machine_create": (C.c_int, [C.POINTER(Config), I32, I32, I32, PP]),
    "tmg_machine_create_shard": (C.c_int, [C.POINTER(Config), I32, I32, I32, I32, I32, PP]),
    "tmg_machine_destroy": (C.c_int, [P]),
    "tmg_machine_info_get": (C.c_int, [P, C.POINTER(MachineInfo)]),
    "tmg_machine_config": (C.c_int, [P, C.POINTER(Config)]),
    "tmg_machine_reset": (C.c_int, [P]),
    "tmg_get_counters": (C.c_int, [P, I32, P]),
    "tmg_set_counters": (C.c_int, [P, I32, P]),
    "tmg_get_include_masks": (C.c_int, [P, I32, P]),
    "tmg_get_include_counts": (C.c_int, [P, I32, P]),
    "tmg_bind_examples": (C.c_int, [P, I64]),
    "tmg_bind_bank": (C.c_int, [P, I32, I64]),
    "tmg_machine_create_devices": (C.c_int, [P, I32, I32, P, I32, P]),
    "tmg_machine_set_windows": (C.c_int, [P, I32]),
    "tmg_last_eval_kernel_ms": (C.c_int, [P, P]),
    "tmg_pool_replica_tallies": (C.c_int, [P, I32, P]),
    "tmg_machine_exchange_info": (C.c_int, [P, P, P]),
    "tmg_nccl_available": (C.c_int, [P, I32]),
    "tmg_comm_unique_id": (C.c_int, [P]),
    "tmg_comm_create": (C.c_int, [P, I32, I32, I32, P]),
    "tmg_comm_destroy": (C.c_int, [P]),
    "tmg_comm_create_ipc": (C.c_int, [I32, I32, I32, I64, P]),
    "tmg_comm_ipc_handle": (C.c_int, [P, P]),
    "tmg_comm_ipc_connect": (C.c_int, [P, P]),
    "tmg_machine_attach_comm": (C.c_int, [P, P]),
    "tmg_bank_bound_examples": (C.c_int, [P, I32, P]),
    "tmg_get_prev_outputs": (C.c_int, [P, I32, P]),
    "tmg_set_prev_outputs": (C.c_int, [P, I32, P]),
    "tmg_pool_create": (C.c_int, [I32, I32, P, P, I64, I32, PP]),
    "tmg_pool_create_device": (C.c_int, [I32, I32, P, P, I64, I32, PP]),
    "tmg_pool_destroy": (C.c_int, [P]),
    "tmg_pool_size": (C.c_int, [P, C.POINTER(I64)]),
    "tmg_pool_get_literals": (C.c_int, [P, P]),
    "tmg_pool_get_tallies": (C.c_int, [P, P]),
    "tmg_pool_set_tallies": (C.c_int, [P, P]),
    "tmg_pool_reset_tallies": (C.c_int, [P]),
    "tmg_pool_tally_device_ptr": (C.c_int, [P, PP]),
    "tmg_pool_delta_device_ptr": (C.c_int, [P, PP]),
    "tmg_pool_tally_ipc_handle": (C.c_int, [P, P]),
    "tmg_pool_set_peers": (C.c_int, [P, P, I32]),
    "tmg_train_epoch": (C.c_int, [P, P, I32, I32, I32, C.POINTER(EpochReportC)]),
    "tmg_train_window": (C.c_int, [P, P, I32, I64, I64, P]),
    "tmg_train_epoch_sequential": (C.c_int, [P, P, I32, C.POINTER(D), P]),
    "tmg_epoch_begin": (C.c_int, [P, P, I32]),
    "tmg_pool_apply_reduced": (C.c_int, [P, P]),
    "tmg_update_clause": (C.c_int, [P, P, I32, I32, P, I64, I64, I64, I32, D, I32, P, P]),
    "tmg_feedback": (C.c_int, [P, I32, I32, P, I32, D, I32, I32, P]),
    "tmg_evaluate_clause": (C.c_int, [P, I32, I32, P, I32, C.POINTER(I32)]),
    "tmg_refresh_tallies": (C.c_int, [P, P]),
    "tmg_class_sums": (C.c_int, [P, P, I32, P]),
    "tmg_predict": (C.c_int, [P, P, P]),
    "tmg_class_sums_literals": (C.c_int, [P, P, I64, I32, P]),
    "tmg_predict_literals": (C.c_int, [P, P, I64, P]),
    "tmg_class_sums_device": (C.c_int, [P, P, I32, P]),
    "tmg_machine_create_regress": (C.c_int, [C.POINTER(Config), I32, I32, PP]),
    "tmg_train_epoch_regress": (C.c_int, [P, P, I32, I32, I32, C.POINTER(EpochReportC)]),
    "tmg_train_epoch_regress_sequential": (C.c_int, [P, P, I32, C.POINTER(D), P]),
    "tmg_regress_predict": (C.c_int, [P, P, P]),
    "tmg_regress_predict_literals": (C.c_int, [P, P, I64, P]),
    "tmg_update_regress": (C.c_int, [P, P, I32, P, P]),
    "tmg_rng_state_init": (None, [U64, U64, P]),
    "tmg_rng_state_next": (U64, [P]),
    "tmg_epoch_order": (C.c_int, [U64, I32, I32, P]),
    "tmg_synth_xor": (C.c_int, [U64, I64, C.c_int, D, C.c_int, P, P]),
    "tmg_synth_mnist": (C.c_int, [U64, C.c_int, C.c_int, D, D, D, I64, I64, P, P, P, P]),
    "tmg_synth_fmnist": (C.c_int, [U64, C.c_int, C.c_int, D, D, C.c_int, D, I64, I64, P, P, P, P]),
    "tmg_synth_imdb": (C.c_int, [U64, C.c_int, C.c_int, D, D, I64, I64, P, P, P, P]),
    "tmg_synth_preset": (C.c_int, [C.c_int, U64, D, I64, I64, P, P, P, P]),
}

_lib = None


def lib():
    """Loads libtmgpu.so (raises if it has not been built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA engine first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class TMError(RuntimeError):
    pass


def check(rc: int):
    """Maps C-ABI status codes to the reference's exception classes."""
    if rc == TMG_OK:
        return
    msg = lib().tmg_last_error().decode(errors="replace")
    if rc == TMG_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == TMG_ERANGE:
        raise IndexError(msg)  # std::out_of_range
    raise TMError(msg)
