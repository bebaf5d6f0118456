"""Pins the C restatement (oracle/tm_oracle.c) against the compiled
reference's golden dumps. CPU only."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_io import EPOCH_CASES, load, manifest


def test_rng_streams():
    nexts, unis = load("rng", "next.npy"), load("rng", "uniform.npy")
    for row, (seed, stream) in enumerate([(42, 0), (42, 3), (7, 123456789)]):
        r = O.Rng(seed, stream)
        assert [r.next() for _ in range(64)] == [int(v) for v in nexts[row]]
        assert [r.uniform() for _ in range(16)] == list(unis[row])
    below = load("rng", "below.npy")
    r = O.Rng(11, 22)
    for row, b in enumerate([1, 2, 3, 10, 1000, 2147483649, 4294967295]):
        assert [r.below(b) for _ in range(8)] == [int(v) for v in below[row]]
    assert np.array_equal(O.Rng(5, 2).shuffled_indices(37), load("rng", "perm37.npy"))
    assert np.array_equal(O.Rng(42, 77).shuffled_indices(1000), load("rng", "perm1000.npy"))


@pytest.mark.parametrize("o", [1, 2, 12, 31, 32, 33, 63, 64, 65, 100, 784])
def test_pack_literals(o):
    bits = load("pack", f"bits_o{o}.npy")
    assert np.array_equal(O.pack_literals(bits), load("pack", f"lits_o{o}.npy"))


def test_gate_probability():
    prob = load("gate", "prob.npy")
    for a, T in enumerate([1, 5, 15, 50]):
        for y in range(2):
            got = [O.clause_update_probability(v, y, T) for v in range(-60, 61)]
            assert got == list(prob[a, y])  # bit-exact doubles


def test_feedback_cases():
    for case in manifest("feedback"):
        k = case["idx"]
        x = load("feedback", f"case{k}_x.npy")
        before = load("feedback", f"case{k}_before.npy")
        after = load("feedback", f"case{k}_after.npy")
        tm = O.Machine(case["o"], 1, 2, case["N"])
        tm.set_counters(before[None])
        lits = O.pack_literals(x)[0]
        out = tm.evaluate(0, 1, lits)
        assert out == case["clause_output"]
        r = O.Rng(case["rng_seed"], case["rng_stream"])
        if case["type"] == 1:
            tm.type_i(0, 1, lits, out, case["s"], case["boost"], r)
        else:
            tm.type_ii(0, 1, lits, out)
        assert np.array_equal(tm.counters[0], after), f"case {k}"
        assert r.next() == int(case["next_draw"])


def _load_state(tag_dir, tag, tm: O.Machine, pool: O.Pool):
    tm.set_counters(load(*tag_dir, f"{tag}_counters.npy"))
    prev = load(*tag_dir, f"{tag}_prev.npy")
    tm.bind(pool.q)
    tm.prev[...] = prev
    pool.tallies[...] = load(*tag_dir, f"{tag}_tallies.npy")


def _check_state(tag_dir, tag, tm: O.Machine, pool: O.Pool):
    assert np.array_equal(tm.counters, load(*tag_dir, f"{tag}_counters.npy"))
    assert np.array_equal(tm.masks, load(*tag_dir, f"{tag}_masks.npy"))
    assert np.array_equal(tm.counts, load(*tag_dir, f"{tag}_counts.npy"))
    assert np.array_equal(tm.prev, load(*tag_dir, f"{tag}_prev.npy"))
    assert np.array_equal(pool.tallies, load(*tag_dir, f"{tag}_tallies.npy"))


def test_update_clause_cases():
    for case in manifest("update_clause"):
        k = case["idx"]
        d = ("update_clause",)
        bits, labels = load(*d, f"case{k}_bits.npy"), load(*d, f"case{k}_labels.npy")
        order = load(*d, f"case{k}_order.npy")
        pool = O.Pool(bits, labels, case["m"])
        tm = O.Machine(case["o"], case["m"], case["n"], case["N"], pool.q)
        _load_state(d, f"case{k}_in", tm, pool)
        r = O.Rng(case["rng_seed"], case["rng_stream"])
        ev = O.update_clause(tm, pool, case["cls"], case["j"], order, case["offset"], case["batch"],
                             case["margin"], case["s"], case["boost"], r)
        assert ev == case["events"]
        _check_state(d, f"case{k}_out", tm, pool)
        assert r.next() == int(case["next_draw"])


@pytest.mark.parametrize("mode", ["epoch_par_w1", "epoch_seq"])
@pytest.mark.parametrize("name", EPOCH_CASES)
def test_epochs(mode, name):
    d = (mode, name)
    man = manifest(*d)
    pool = O.Pool(load(*d, "train_x.npy"), load(*d, "train_y.npy"), man["m"])
    tm = O.Machine(man["o"], man["m"], man["n"], man["N"], pool.q)
    for ep in man["epochs"]:
        e = ep["epoch"]
        if mode == "epoch_par_w1":
            ev = O.train_epoch_parallel(tm, pool, man["margin"], man["s"], man["boost"], man["seed"], 1, e)
            _check_state(d, f"epoch{e}", tm, pool)
        else:
            ev = O.train_epoch_sequential(tm, pool, man["margin"], man["s"], man["boost"], man["seed"], e)
            assert np.array_equal(tm.counters, load(*d, f"epoch{e}_counters.npy"))
        assert [int(v) for v in ev] == ep["feedback_events"]
    test_lits = O.pack_literals(load(*d, "test_x.npy"))
    assert np.array_equal(tm.class_sums(test_lits), load(*d, "test_sums.npy"))
    assert np.array_equal(tm.predict(test_lits), load(*d, "test_pred.npy"))
    if mode == "epoch_par_w1":
        O.refresh_tallies(tm, pool)
        _check_state(d, "refreshed", tm, pool)


@pytest.mark.parametrize("mode", ["par", "seq"])
def test_regression_head(mode):
    man = manifest("regression")
    x, y = load("regression", "train_x.npy"), load("regression", "train_y.npy")
    pool = O.Pool(x, y, 1)  # scaled targets == y here (T = y_max - y_min = 10)
    tm = O.Machine(man["o"], 1, man["clauses"], man["N"], pool.q)
    T_, s, seed = man["margin"], man["s"], man["seed"]
    for e, want in enumerate(man[f"{mode}_events"]):
        if mode == "par":
            ev = O.train_epoch_regress_parallel(tm, pool, T_, s, False, seed, 1, e)
            assert np.array_equal(pool.tallies[:, 0], load("regression", f"par_epoch{e}_tallies.npy"))
            assert np.array_equal(tm.prev[0].reshape(-1), load("regression", f"par_epoch{e}_prev.npy"))
        else:
            ev = O.train_epoch_regress_sequential(tm, pool, T_, s, False, seed, e)
        assert ev == want
        assert np.array_equal(tm.counters[0], load("regression", f"{mode}_epoch{e}_counters.npy"))
    tx = load("regression", "test_x.npy")
    pred = O.predict_scaled(tm, O.pack_literals(tx), T_)
    assert np.array_equal(pred, load("regression", f"{mode}_predict_scaled.npy"))
    if mode == "seq":
        r = O.Rng(99, 4)
        assert O.update_regress(tm, O.pack_literals(tx[3])[0], 7, T_, s, False, r) == man["update_regress_events"]
        assert np.array_equal(tm.counters[0], load("regression", "update_regress_counters.npy"))
        assert r.next() == int(man["update_regress_next"])


@pytest.mark.parametrize("name,o,m,n", [("mnist_rand", 784, 10, 50), ("single_bank", 30, 1, 8),
                                        ("dense_o64", 64, 3, 12)])
def test_inference_random_states(name, o, m, n):
    bits = load("inference", f"{name}_bits.npy")
    tm = O.Machine(o, m, n, 128)
    tm.set_counters(load("inference", f"{name}_counters.npy"))
    lits = O.pack_literals(bits)
    assert np.array_equal(tm.class_sums(lits), load("inference", f"{name}_sums.npy"))
    assert np.array_equal(tm.predict(lits), load("inference", f"{name}_pred.npy"))
    pool = O.Pool(bits, np.zeros(bits.shape[0], np.int32), m)
    O.refresh_tallies(tm, pool)
    assert np.array_equal(pool.tallies, load("inference", f"{name}_tallies.npy"))
    assert np.array_equal(tm.prev, load("inference", f"{name}_prev.npy"))


def test_philox_known_answers():
    """The async engine's generator, restated in oracle/tm_oracle_async.c, on
    the Random123 published known-answer vectors (kat_vectors, philox4x32 R=10)."""
    assert list(O.philox4x32([0, 0, 0, 0], 0, 0, 10)) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    ff = 0xFFFFFFFF
    assert list(O.philox4x32([ff] * 4, ff, ff, 10)) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    pi = [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344]
    assert list(O.philox4x32(pi, 0xA4093822, 0x299F31D0, 10)) == [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_async_type_i_restatement_rates():
    """The restated async draw feeds back at p_low = 1/s with clause output 0
    (Table 1): pooled over many examples, within binomial noise."""
    o, N, s = 64, 128, 10.0
    counters = np.full(2 * o, 100, np.uint16)
    lits = O.pack_literals(np.zeros(o, np.uint8))[0]
    moved = 0
    trials = 400
    for i in range(trials):
        after = O.async_type_i(counters, lits, o, N, 0, s, False, 5, i, 1, 0, 1)
        moved += int((after != counters).sum())
    rate = moved / (trials * 2 * o)
    assert abs(rate - 0.1) < 0.006, rate
