"""B200-native asynchronous clause-parallel Tsetlin Machine (arXiv 2009.04861).

Host API mirroring the reference's C++ API (tsetlin::TMConfig, MultiClassTM,
ExamplePool, train_epoch_parallel, train_epoch_sequential, classify,
predict_all, export_vote_sums, refresh_tallies, update_clause, feedback,
RegressionHead, tmmodel v1 I/O) over the C ABI of libtmgpu.so
(include/tmgpu.h), whose kernels are hand-written for sm_100a.

Importing the package loads libtmgpu.so and raises ImportError if it has not
been built: there is no CPU fallback.
"""
import importlib.util as _ilu
import os as _os

# Sharded machines load NCCL at run time (csrc/group.cu). Point the engine at
# the NCCL wheel torch links against, so that a process which uses the
# engine's NCCL before importing torch does not leave an older system
# libnccl.so.2 in place for libtorch_cuda.so to bind to.
if "TMG_NCCL_LIB" not in _os.environ:
    _spec = _ilu.find_spec("nvidia.nccl") if _ilu.find_spec("nvidia") else None
    for _root in (_spec.submodule_search_locations or []) if _spec else []:
        _cand = _os.path.join(_root, "lib", "libnccl.so.2")
        if _os.path.exists(_cand):
            _os.environ["TMG_NCCL_LIB"] = _cand
            break

from . import _capi as _capi_mod  # noqa: E402

_capi_mod.lib()  # fail loudly at import when the CUDA engine is missing

from .model_io import load_model_file, save_model_file  # noqa: E402
from .tsetlin import (MODE_ASYNC, MODE_AUTO, MODE_SYNC_MIRROR, PREDICT, TRAIN, ClassBank, Comm, EpochReport,  # noqa: E402
                      ExamplePool, MultiClassTM, RegressionHead, Rng, TMConfig, class_sums, classify,
                      device_count, epoch_order, evaluate_accuracy, nccl_available, evaluate_clause, evaluate_scaled_mae,
                      export_vote_sums, feedback_rates, literal_words, predict_all, predict_literals,
                      predict_regress, predict_scaled, predict_scaled_all, refresh_tallies,
                      train_epoch_parallel, train_epoch_regress_parallel, train_epoch_regress_sequential,
                      train_epoch_sequential, type_i_feedback, type_ii_feedback, update_clause,
                      update_regress, vote_sum)

__all__ = [
    "MODE_ASYNC", "MODE_AUTO", "MODE_SYNC_MIRROR", "PREDICT", "TRAIN", "ClassBank", "Comm", "EpochReport",
    "ExamplePool", "MultiClassTM", "RegressionHead", "Rng", "TMConfig", "class_sums", "classify",
    "device_count", "epoch_order", "evaluate_accuracy", "nccl_available", "evaluate_clause", "evaluate_scaled_mae",
    "export_vote_sums", "feedback_rates", "literal_words", "load_model_file", "predict_all",
    "predict_literals", "predict_regress", "predict_scaled", "predict_scaled_all", "refresh_tallies",
    "save_model_file", "train_epoch_parallel", "train_epoch_regress_parallel",
    "train_epoch_regress_sequential", "train_epoch_sequential", "type_i_feedback", "type_ii_feedback",
    "update_clause", "update_regress", "vote_sum",
]
