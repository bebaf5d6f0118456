"""B200-native asynchronous clause-parallel Tsetlin Machine (arXiv 2009.04861).

Host API mirroring the reference's C++ API (tsetlin::TMConfig, MultiClassTM,
ExamplePool, train_epoch_parallel, train_epoch_sequential, classify,
predict_all, export_vote_sums, refresh_tallies, update_clause, feedback) over
the C ABI of libtmgpu.so (include/tmgpu.h), whose kernels are hand-written for
sm_100a.
"""
from .tsetlin import (MODE_ASYNC, MODE_SYNC_MIRROR, PREDICT, TRAIN, ClassBank, EpochReport,
                      ExamplePool, MultiClassTM, Rng, TMConfig, class_sums, classify, device_count,
                      epoch_order, evaluate_accuracy, evaluate_clause, export_vote_sums,
                      feedback_rates, literal_words, predict_all, predict_literals, refresh_tallies,
                      train_epoch_parallel, train_epoch_sequential, type_i_feedback,
                      type_ii_feedback, update_clause, vote_sum)

__all__ = [
    "MODE_ASYNC", "MODE_SYNC_MIRROR", "PREDICT", "TRAIN", "ClassBank", "EpochReport",
    "ExamplePool", "MultiClassTM", "Rng", "TMConfig", "class_sums", "classify", "device_count",
    "epoch_order", "evaluate_accuracy", "evaluate_clause", "export_vote_sums", "feedback_rates",
    "literal_words", "predict_all", "predict_literals", "refresh_tallies", "train_epoch_parallel",
    "train_epoch_sequential", "type_i_feedback", "type_ii_feedback", "update_clause", "vote_sum",
]
