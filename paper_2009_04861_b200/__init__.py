"""B200-native asynchronous clause-parallel Tsetlin Machine (arXiv 2009.04861).

Host API mirroring the reference's C++ API (tsetlin::TMConfig, MultiClassTM,
ExamplePool, train_epoch_parallel, train_epoch_sequential, classify,
predict_all, export_vote_sums, refresh_tallies, update_clause, feedback,
RegressionHead, tmmodel v1 I/O) over the C ABI of libtmgpu.so
(include/tmgpu.h), whose kernels are hand-written for sm_100a.

Importing the package loads libtmgpu.so and raises ImportError if it has not
been built: there is no CPU fallback.
"""
from . import _capi as _capi_mod

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
