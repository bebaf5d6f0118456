"""CPU-only checks of the boundary: libtmgpu.so loads and exports every
symbol include/*.h declares; host-side logic (config validation, RNG streams,
synthetic data, sharding arithmetic) matches the reference/oracle."""
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(REPO, "paper_2009_04861_b200", "_lib", "libtmgpu.so")


def _declared(header):
    src = open(os.path.join(REPO, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(tmg_\w+)\s*\(", src, flags=re.M))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build first: make -C paper_2009_04861_b200/csrc"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    declared = _declared("tmgpu.h")
    assert len(declared) > 40
    missing = sorted(declared - exported)
    assert not missing, f"declared but not exported: {missing}"


def test_ctypes_signatures_cover_header():
    from paper_2009_04861_b200 import _capi
    assert set(_capi.SIGNATURES) == _declared("tmgpu.h")
    _capi.lib()  # every signature resolves


def test_config_validation_matches_reference():
    import paper_2009_04861_b200 as T
    T.TMConfig().validate()
    for bad, msg in [(dict(clauses=3), "even"), (dict(clauses=0), "even"), (dict(margin=0), "margin"),
                     (dict(specificity=0.5), "specificity"), (dict(state_depth=0), "state depth"),
                     (dict(state_depth=16384), "too large"), (dict(epochs=-1), "epochs"),
                     (dict(workers=-1), "workers")]:
        with pytest.raises(ValueError, match=msg):
            T.TMConfig(**bad).validate()


def test_host_rng_and_epoch_order_match_oracle():
    import paper_2009_04861_b200 as T
    for seed, stream in [(42, 0), (7, 123456789), (2**63 + 5, 3)]:
        a, b = T.Rng(seed, stream), O.Rng(seed, stream)
        assert [a.next() for _ in range(50)] == [b.next() for _ in range(50)]
    for e in range(3):
        want = O.Rng(42, O.mix_stream(2, e)).shuffled_indices(1000)
        assert np.array_equal(T.epoch_order(42, e, 1000), want)


def test_synth_matches_reference_driver_data():
    """The generators are shared with oracle/_ref; golden epoch fixtures were
    trained on them."""
    from paper_2009_04861_b200 import synth
    from tests.golden_io import load
    d = synth.make("xor", 100, 60, 7, 0.1)
    assert np.array_equal(d.train_x, load("epoch_par_w1", "xor12", "train_x.npy"))
    assert np.array_equal(d.train_y, load("epoch_par_w1", "xor12", "train_y.npy"))
    assert np.array_equal(d.test_x, load("epoch_par_w1", "xor12", "test_x.npy"))
    m = synth.make("mnist", 100, 60, 2009)
    assert np.array_equal(m.train_x, load("epoch_par_w1", "mnist_small", "train_x.npy"))
    assert np.array_equal(m.test_y, load("epoch_par_w1", "mnist_small", "test_y.npy"))
    # MNIST recipe is non-saturating: classes balanced-ish, density ~0.2-0.4
    assert 0.15 < m.train_x.mean() < 0.45


def test_model_file_parser_matches_reference_text():
    """tmmodel v1 written by the reference parses to its counters (f3)."""
    from paper_2009_04861_b200 import model_io
    from tests.golden_io import GOLDEN, load
    text = open(os.path.join(GOLDEN, "models", "xor12_model.txt")).read()
    p = model_io.parse(text)
    assert p["task"] == "classify" and p["features"] == 12 and p["classes"] == 2
    assert p["config"].specificity == 3.9 and p["config"].clauses == 20
    want = load("epoch_par_w1", "xor12", "epoch3_counters.npy")
    for c in range(2):
        assert np.array_equal(p["banks"][c], want[c])
    r = model_io.parse(open(os.path.join(GOLDEN, "regression", "regress_model.txt")).read())
    assert r["task"] == "regress" and r["range"] == (0.0, 10.0)
    with pytest.raises(RuntimeError, match="not a tmmodel"):
        model_io.parse("hello v1")
    with pytest.raises(RuntimeError, match="end marker"):
        model_io.parse(text.replace("end\n", "fin\n"))


def test_bench_csv_schema_matches_reference():
    """f4: the reference's CSV columns and %.9g formatting (bench.cpp:120-142)."""
    from paper_2009_04861_b200.bench_sweep import (BenchRecord, median_epoch_seconds, read_bench_csv,
                                                   write_bench_csv)
    recs = [BenchRecord("par", 64, 2000, 0, 0.1234567891234, "accuracy", 0.9375),
            BenchRecord("par", 64, 2000, 1, 0.2, "accuracy", 1.0),
            BenchRecord("par", 64, 2000, 2, 0.05, "accuracy", 0.5)]
    text = write_bench_csv(recs)
    assert text.splitlines()[0] == "mode,workers,clauses,epoch,seconds,metric_name,metric_value"
    assert text.splitlines()[1] == "par,64,2000,0,0.123456789,accuracy,0.9375"
    assert median_epoch_seconds(recs, "par", 2000) == pytest.approx(0.1234567891234)
    assert [r.epoch for r in read_bench_csv(text)] == [0, 1, 2]
    with pytest.raises(ValueError):
        median_epoch_seconds(recs, "seq", 2000)


def test_shard_ranges_even_aligned_and_cover():
    from paper_2009_04861_b200.distributed import shard_range, window_bounds
    for n in [2, 20, 2000, 2002, 7000]:
        for world in [1, 2, 3, 4, 8]:
            if n // 2 < world:
                continue
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, _) in zip(spans, spans[1:]):
                assert b == c
            assert all(a % 2 == 0 and b % 2 == 0 and b > a for a, b in spans)
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 2
    assert window_bounds(10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert window_bounds(5, 9) == [(k, k + 1) for k in range(5)]


def test_host_companions_match_reference(tmp_path):
    """data_io.hpp / metrics.hpp / bench CSV of the drop-in (csrc/facade_data.cpp,
    host code, no GPU): tests/cpp/data_driver.cpp "host" — generators, dense
    binary and CSV files with their error messages, the binarizer (fit, apply,
    tmbinarizer v1 round trip), metrics, bench CSV — prints the reference's
    transcript (tests/golden/data_driver_host_ref.txt) line for line."""
    import subprocess
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    drv = os.path.join(repo, "paper_2009_04861_b200", "_lib", "data_driver_gpu")
    out = subprocess.run([drv, "host", str(tmp_path)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    want = [l for l in open(os.path.join(repo, "tests", "golden", "data_driver_host_ref.txt")).read().splitlines()
            if l.strip()]
    got = [l for l in out.stdout.splitlines() if l.strip()]
    assert got == want


def _cli_golden(part):
    lines = open(os.path.join(REPO, "tests", "golden", "cli_session_ref.txt")).read().splitlines()
    from tests.cli_session import HOST
    # the host part is the transcript up to the first command of the gpu part
    n_host = [i for i, l in enumerate(lines) if l.startswith("$ ")][len(HOST)]
    return lines[:n_host] if part == "host" else lines


def test_cli_host_part_matches_reference():
    """The `tm` command line (f4, cli.cpp:429-530) without a GPU: synth files,
    parse failures with CLI11's exit codes, validation errors, missing files
    (exit 2) — the same transcript as our CLI source linked with the reference
    library (tests/golden/cli_session_ref.txt)."""
    from tests.cli_session import run
    tm = os.path.join(REPO, "paper_2009_04861_b200", "_lib", "tm")
    assert os.path.exists(tm), "build first: make -C paper_2009_04861_b200/csrc"
    assert run(tm, "host") == _cli_golden("host")


def test_xoshiro_jump_ahead_matches_stepping():
    """The GF(2) jump matrices behind the bit-exact parallel replays
    (engine.cu gf2_pow; applied on the GPU by sequential.cu / train.cu
    draw_type_i_bits): M^k applied to a state equals k steps of rng.hpp
    next() — for the chunk and 2o distances of the configs' shapes."""
    import ctypes as C

    import paper_2009_04861_b200 as T
    from paper_2009_04861_b200._capi import check, lib
    for k in (1, 2, 49, 147, 625, 1568, 4704, 20000):
        r = T.Rng(2009, k)
        jumped = r.state.copy()
        check(lib().tmg_debug_xoshiro_jump(C.c_void_p(jumped.ctypes.data), k))
        for _ in range(k):
            r.next()
        assert np.array_equal(jumped, r.state), k
