"""The reference's own acceptance criteria run against the
B200 engine, on the reference's own synthetic generators (written by the `tm`
command line, `tm synth`, which is the reference's data_io code path
restated and transcript-checked in tests/cli_session.py).

  3  XOR convergence            test_xor_convergence
  4  parallel/sequential parity test_parallel_sequential_parity
  7  scaling shape              test_scaling_shape
  9  determinism                test_determinism_model_files
  1  Table-1 conformance        test_gpu_async.py::test_type_i_table1_conformance (s = 1.5, 4, 15 included)
  2  gating                     test_gpu_async.py::test_async_gate_zero_at_margin + the bit-exact replays
  5  eventual consistency       test_gpu_async.py (refresh vs brute force on trained/random states)
  6  lost-update freedom        test_gpu_async.py::test_async_contended_tallies_lose_no_update
  8  regression (optional)      not asserted: the reference itself does not reach the staircase bar
                                (DESIGN.md §2); regression parity is bit-exact (test_gpu_regression.py)

"parallel (W=8)" is the asynchronous all-clause GPU trainer; "sequential" is
train_epoch_sequential replayed bit-exactly on the GPU."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

T = pytest.importorskip("paper_2009_04861_b200")
from paper_2009_04861_b200 import model_io  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TM = os.path.join(REPO, "paper_2009_04861_b200", "_lib", "tm")


def _synth(tmp, name, train, test, seed, **kw):
    """tm synth → (train_x, train_y, test_x, test_y) from the dense binary files."""
    out = str(tmp / f"{name}{seed}")
    args = [TM, "synth", "--name", name, "--train", str(train), "--test", str(test), "--seed", str(seed),
            "--out", out]
    for k, v in kw.items():
        args += [f"--{k}", str(v)]
    subprocess.run(args, check=True, capture_output=True)
    a = np.loadtxt(out + ".train", dtype=np.int64, ndmin=2)
    b = np.loadtxt(out + ".test", dtype=np.int64, ndmin=2)
    return (a[:, :-1].astype(np.uint8), a[:, -1].astype(np.int32), b[:, :-1].astype(np.uint8),
            b[:, -1].astype(np.int32))


def _machine(x, y, m, clauses, margin, s, seed):
    cfg = T.TMConfig(clauses=clauses, margin=margin, specificity=s, seed=seed)
    return T.MultiClassTM(cfg, x.shape[1], m), T.ExamplePool(x.shape[1], x, y, m)


def _train(tm, pool, epochs, parallel, stop_at=None):
    for e in range(epochs):
        if parallel:
            T.train_epoch_parallel(tm, pool, 8, e)
        else:
            T.train_epoch_sequential(tm, pool, e)
        if stop_at is not None and T.evaluate_accuracy(tm, pool) >= stop_at:
            return e + 1
    return epochs


@pytest.mark.parametrize("parallel", [False, True])
def test_xor_convergence(tmp_path, parallel):
    """Criterion 3: noise-free XOR (q = 1000), n = 10, T = 5, s = 3 -> 100 %
    train accuracy within 50 epochs on 5/5 seeds."""
    for seed in range(1, 6):
        x, y, _, _ = _synth(tmp_path, "xor", 1000, 200, seed)
        tm, pool = _machine(x, y, 2, 10, 5, 3.0, seed)
        used = _train(tm, pool, 50, parallel, stop_at=1.0)
        assert T.evaluate_accuracy(tm, pool) == 1.0, (seed, parallel, used)


def _mean_test_acc(tmp, name, data_kw, m, clauses, margin, s, epochs, parallel):
    accs = []
    for seed in range(1, 6):
        x, y, tx, ty = _synth(tmp, name, data_kw["q"], data_kw["qt"], seed, **data_kw["extra"])
        tm, pool = _machine(x, y, m, clauses, margin, s, seed)
        _train(tm, pool, epochs, parallel)
        accs.append(T.evaluate_accuracy(tm, T.ExamplePool(tx.shape[1], tx, ty, m)))
    return float(np.mean(accs)), accs


@pytest.mark.parametrize("name,data_kw,m,clauses,margin,s,epochs", [
    ("xor", {"q": 5000, "qt": 5000, "extra": {"noise": 0.1}}, 2, 10, 5, 3.0, 20),
    ("patterns", {"q": 2000, "qt": 1000, "extra": {"noise": 0.1, "classes": 4, "zone": 5}}, 4, 40, 15, 3.9, 15),
])
def test_parallel_sequential_parity(tmp_path, name, data_kw, m, clauses, margin, s, epochs):
    """Criterion 4: noisy XOR (10 % noise, q = 5000) and the 20-feature /
    4-class clause-pattern data: |mean test accuracy(parallel) -
    mean(sequential)| <= 2 points over 5 seeds."""
    seq, seq_all = _mean_test_acc(tmp_path, name, data_kw, m, clauses, margin, s, epochs, False)
    par, par_all = _mean_test_acc(tmp_path, name, data_kw, m, clauses, margin, s, epochs, True)
    print(f"{name}: sequential {seq:.4f} {seq_all}  parallel {par:.4f} {par_all}")
    assert abs(par - seq) <= 0.02, (seq, par)


def test_scaling_shape(tmp_path):
    """Criterion 7: sequential seconds/epoch grows at most x2.6 per clause
    doubling over n = 160 ... 1280, and the parallel epoch at n = 2048 takes
    <= 0.5x the sequential one (on the GPU: far less). The criterion's lower
    bound (x1.6, the CPU trainer's linear cost) is not asserted: the GPU
    replay of the sequential trainer applies the gated clauses of an example
    in parallel, so it grows sub-linearly (x1.44 / 1.64 / 1.89 measured; the
    serial replay, TMG_SEQ_SERIAL=1: x1.68 / 1.68 / 2.15)."""
    x, y, _, _ = _synth(tmp_path, "patterns", 1000, 10, 7, classes=4, zone=5)

    def seconds(n, parallel):
        tm, pool = _machine(x, y, 4, n, 15, 3.9, 7)
        _train(tm, pool, 1, parallel)  # warm-up epoch, then the timed one
        rep = (T.train_epoch_parallel(tm, pool, 8, 1) if parallel else T.train_epoch_sequential(tm, pool, 1))
        return rep.seconds

    seq = [seconds(n, False) for n in (160, 320, 640, 1280)]
    growth = [b / a for a, b in zip(seq, seq[1:])]
    print(f"sequential s/epoch {seq}, growth per doubling {growth}")
    assert all(1.0 < g <= 2.6 for g in growth), growth
    s2048, p2048 = seconds(2048, False), seconds(2048, True)
    print(f"n=2048: sequential {s2048:.4f} s, parallel {p2048:.6f} s")
    assert p2048 <= 0.5 * s2048


@pytest.mark.parametrize("parallel_w1", [False, True])
def test_determinism_model_files(tmp_path, parallel_w1):
    """Criterion 9: sequential and W = 1 parallel runs with fixed seeds are
    bit-identical across repeated invocations (model files compare equal)."""
    x, y, _, _ = _synth(tmp_path, "patterns", 600, 10, 3, classes=4, zone=5, noise=0.1)
    texts = []
    for _ in range(2):
        tm, pool = _machine(x, y, 4, 20, 10, 3.9, 11)
        for e in range(3):
            if parallel_w1:
                T.train_epoch_parallel(tm, pool, 1, e, mode=T.MODE_SYNC_MIRROR)
            else:
                T.train_epoch_sequential(tm, pool, e)
        texts.append(model_io.dumps(tm))
    assert texts[0] == texts[1]
