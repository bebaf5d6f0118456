"""Regression head and tmmodel v1 files (f3) on the GPU
against the compiled reference's golden dumps (tests/golden/regression,
tests/golden/models)."""
import json
import os

import numpy as np
import pytest

from tests.golden_io import GOLDEN, load

pytestmark = pytest.mark.gpu

T = pytest.importorskip("paper_2009_04861_b200")
from paper_2009_04861_b200 import model_io, tsetlin as TS  # noqa: E402


def _man():
    return json.load(open(os.path.join(GOLDEN, "regression", "manifest.json")))


def _head(man):
    cfg = T.TMConfig(clauses=man["clauses"], margin=man["margin"], specificity=man["s"], state_depth=man["N"],
                     seed=man["seed"])
    return TS.RegressionHead(cfg, man["o"], man["y_min"], man["y_max"])


@pytest.mark.parametrize("mode", ["par", "seq"])
def test_regression_epochs_bit_exact(mode):
    man = _man()
    head = _head(man)
    x, y = load("regression", "train_x.npy"), load("regression", "train_y.npy")
    pool = TS.regress_pool(head, x, y)
    for e, want in enumerate(man[f"{mode}_events"]):
        if mode == "par":
            rep = TS.train_epoch_regress_parallel(head, pool, 1, e, mode=T.MODE_SYNC_MIRROR)
        else:
            rep = TS.train_epoch_regress_sequential(head, pool, e)
        assert rep.feedback_events == [want], f"epoch {e}"
        assert np.array_equal(head.bank.counters(), load("regression", f"{mode}_epoch{e}_counters.npy"))
        if mode == "par":
            assert np.array_equal(pool.tallies()[:, 0], load("regression", f"par_epoch{e}_tallies.npy"))
            assert np.array_equal(head.bank.prev_outputs().reshape(-1), load("regression", f"par_epoch{e}_prev.npy"))
    tx, ty = load("regression", "test_x.npy"), load("regression", "test_y.npy")
    test = T.ExamplePool(man["o"], tx, ty, 1)
    pred = TS.predict_scaled_all(head, test)
    assert np.array_equal(pred, load("regression", f"{mode}_predict_scaled.npy"))
    assert TS.evaluate_scaled_mae(head, test) == pytest.approx(man[f"{mode}_mae"], abs=0)
    if mode == "seq":
        from oracle import oracle as O
        r = T.Rng(99, 4)
        ev = TS.update_regress(head, O.pack_literals(tx[3])[0], 7.0, r)
        assert ev == man["update_regress_events"]
        assert np.array_equal(head.bank.counters(), load("regression", "update_regress_counters.npy"))
        assert r.next() == int(man["update_regress_next"])
        want = open(os.path.join(GOLDEN, "regression", "regress_model.txt")).read()
        assert model_io.dumps(head) == want


def test_regression_async_learns():
    man = _man()
    head = _head(man)
    x, y = load("regression", "train_x.npy"), load("regression", "train_y.npy")
    pool = TS.regress_pool(head, x, y)
    for e in range(30):
        TS.train_epoch_regress_parallel(head, pool, 8, e)
    tx, ty = load("regression", "test_x.npy"), load("regression", "test_y.npy")
    mae = TS.evaluate_scaled_mae(head, T.ExamplePool(man["o"], tx, ty, 1))
    assert mae < 2.5, mae  # reference W=1, 3 epochs: 2.12; a constant predictor: ~1.9-2.5


def test_bench_sweep_csv_gpu():
    """f4: the reference's clause sweep (bench.cpp:45-118) with GPU rows."""
    from paper_2009_04861_b200 import bench_sweep as BS
    from paper_2009_04861_b200 import synth
    d = synth.make("xor", 2000, 500, 7, 0.1)
    opts = BS.BenchOptions(clause_counts=[10, 20], modes=["seq", "par"], warmup_epochs=1, measured_epochs=2)
    recs = BS.bench_sweep(d.train_x, d.train_y, d.test_x, d.test_y,
                          T.TMConfig(margin=15, specificity=3.9, seed=1), opts)
    assert len(recs) == 2 * 2 * 2
    assert all(r.metric_name == "accuracy" and 0.4 <= r.metric_value <= 1.0 and r.seconds > 0 for r in recs)
    text = BS.write_bench_csv(recs)
    assert len(text.splitlines()) == 9
    assert BS.median_epoch_seconds(recs, "par", 20) > 0


def test_model_files_roundtrip_and_match_reference():
    """tmmodel v1: GPU-trained (sync mirror) machine == reference bytes; load back."""
    d = ("epoch_par_w1", "xor12")
    x, y = load(*d, "train_x.npy"), load(*d, "train_y.npy")
    tm = T.MultiClassTM(T.TMConfig(clauses=20, margin=15, specificity=3.9, seed=1), 12, 2)
    pool = T.ExamplePool(12, x, y, 2)
    for e in range(4):
        T.train_epoch_parallel(tm, pool, 1, e, mode=T.MODE_SYNC_MIRROR)
    text = model_io.dumps(tm)
    assert text == open(os.path.join(GOLDEN, "models", "xor12_model.txt")).read()
    back = model_io.loads(text)
    for c in range(2):
        assert np.array_equal(back.banks[c].counters(), tm.banks[c].counters())
    with pytest.raises(RuntimeError, match="outside"):
        model_io.loads(text.replace("\n135 ", "\n999 ", 1))
    head = model_io.loads(open(os.path.join(GOLDEN, "regression", "regress_model.txt")).read())
    assert isinstance(head, TS.RegressionHead) and head.config.margin == 10
