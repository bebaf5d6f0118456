"""The drop-in check: tests/cpp/api_driver.cpp, written only against the
reference's public C++ API, is compiled once against the reference (CPU,
oracle/_ref/api_driver_ref; transcript in tests/golden/api_driver_ref.txt)
and once against include/tsetlin/*.hpp + libtsetlin_b200.so (GPU). Every
deterministic result must be identical."""
import os
import subprocess

import numpy as np
import pytest

from tests.golden_io import EPOCH_CASES, GOLDEN, load, manifest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GPU_DRIVER = os.path.join(REPO, "paper_2009_04861_b200", "_lib", "api_driver_gpu")
REF_DRIVER = os.path.join(REPO, "oracle", "_ref", "api_driver_ref")


DET_ENV = dict(os.environ, TSETLIN_DETERMINISTIC="1")


def _lines(text):
    return [l for l in text.splitlines() if l.strip()]


def test_same_source_driver_matches_reference():
    assert os.path.exists(GPU_DRIVER), "build first (make -C paper_2009_04861_b200/csrc)"
    # the transcript includes one-worker train_epoch_parallel epochs: the
    # bit-exact replay is selected by TSETLIN_DETERMINISTIC=1 (TMG_MODE_AUTO)
    gpu = subprocess.run([GPU_DRIVER], capture_output=True, text=True, timeout=600, env=DET_ENV)
    assert gpu.returncode == 0, gpu.stderr
    want = _lines(open(os.path.join(GOLDEN, "api_driver_ref.txt")).read())
    if os.path.exists(REF_DRIVER):  # the live reference binary, when it travelled
        want = _lines(subprocess.run([REF_DRIVER], capture_output=True, text=True, check=True).stdout)
    got = _lines(gpu.stdout)
    diffs = [(w, g) for w, g in zip(want, got) if w != g]
    assert len(got) == len(want) and not diffs, f"first differences: {diffs[:5]}"


def test_same_source_bench_sweep_matches_reference():
    """bench.hpp's bench_sweep (f4) on the GPU trainers: tests/cpp/data_driver.cpp
    "bench" (seq and one-worker par, classification and regression) prints the
    reference's records (seconds excluded) line for line."""
    drv = os.path.join(REPO, "paper_2009_04861_b200", "_lib", "data_driver_gpu")
    out = subprocess.run([drv, "bench"], capture_output=True, text=True, timeout=600, env=DET_ENV)
    assert out.returncode == 0, out.stderr
    want = _lines(open(os.path.join(GOLDEN, "data_driver_bench_ref.txt")).read())
    got = _lines(out.stdout)
    diffs = [(w, g) for w, g in zip(want, got) if w != g]
    assert len(got) == len(want) and not diffs, f"first differences: {diffs[:5]}"


@pytest.mark.parametrize("name", EPOCH_CASES)
def test_sequential_trainer_bit_exact(name):
    """train_epoch_sequential (f1) replayed on the GPU == the reference."""
    import paper_2009_04861_b200 as T
    d = ("epoch_seq", name)
    man = manifest(*d)
    pool = T.ExamplePool(man["o"], load(*d, "train_x.npy"), load(*d, "train_y.npy"), man["m"])
    cfg = T.TMConfig(clauses=man["n"], margin=man["margin"], specificity=man["s"], state_depth=man["N"],
                     boost_true_positive=bool(man["boost"]), seed=man["seed"])
    tm = T.MultiClassTM(cfg, man["o"], man["m"])
    for ep in man["epochs"]:
        e = ep["epoch"]
        rep = T.train_epoch_sequential(tm, pool, e)
        assert rep.feedback_events == ep["feedback_events"], f"events epoch {e}"
        counters = load(*d, f"epoch{e}_counters.npy")
        for c in range(man["m"]):
            assert np.array_equal(tm.banks[c].counters(), counters[c]), f"epoch {e} bank {c}"
    test = T.ExamplePool(man["o"], load(*d, "test_x.npy"), load(*d, "test_y.npy"), man["m"])
    assert np.array_equal(T.class_sums(tm, test), load(*d, "test_sums.npy"))
    assert np.array_equal(T.predict_all(tm, test), load(*d, "test_pred.npy"))


def test_cli_session_matches_reference():
    """The `tm` command line (f4, cli.cpp:429-530) on the GPU facade: train
    (seq, one-worker par, TM_THREADS override, classify and regress, dense and
    CSV input with the binarizer), eval of the saved models, bench CSV — every
    stdout line and every written file (seconds masked) identical to the same
    CLI source linked with the reference library."""
    from tests.cli_session import run
    from tests.test_cpu_boundary import _cli_golden
    tm = os.path.join(REPO, "paper_2009_04861_b200", "_lib", "tm")
    want = _cli_golden("all")
    ref = os.path.join(REPO, "oracle", "_ref", "tm_ref")
    if os.path.exists(ref):
        want = run(ref, "all")
    got = run(tm, "all")
    diffs = [(w, g) for w, g in zip(want, got) if w != g]
    assert len(got) == len(want) and not diffs, f"first differences: {diffs[:5]}"


def test_cli_parallel_mode_trains(tmp_path):
    """`tm train --mode par --workers 8`: the asynchronous all-clause trainer
    behind the command line (not a replay); learns the synthetic patterns."""
    tm = os.path.join(REPO, "paper_2009_04861_b200", "_lib", "tm")
    env = {k: v for k, v in os.environ.items() if k != "TM_THREADS"}
    p = subprocess.run([tm, "train", "--synth", "patterns", "--synth-train", "2000", "--synth-test", "500",
                        "--classes", "4", "--clauses", "40", "--epochs", "5", "--mode", "par", "--workers", "8",
                        "--report", str(tmp_path / "r.csv"), "--out", str(tmp_path / "m.model")],
                       capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, p.stderr
    vals = dict(l.split(" ", 1) for l in p.stdout.splitlines() if " " in l)
    assert float(vals["test_accuracy"]) >= 0.9, p.stdout
    rows = open(tmp_path / "r.csv").read().splitlines()
    assert rows[0] == "mode,workers,clauses,epoch,seconds,metric_name,metric_value"
    assert len(rows) == 1 + 2 * 5 and all(r.startswith("par,8,40,") for r in rows[1:])
    e = subprocess.run([tm, "eval", "--model", str(tmp_path / "m.model"), "--data", str(tmp_path / "m.model")],
                       capture_output=True, text=True, timeout=120, env=env)
    assert e.returncode == 1  # a model file is not a dataset: the loader's runtime_error -> exit 1
