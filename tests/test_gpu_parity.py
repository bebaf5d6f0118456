"""GPU parity: the sm_100a engine (through the C ABI) against the reference's
golden dumps (tests/golden/, from the compiled reference) and the oracle.

Bit-exact for everything deterministic: packing, class sums / predictions on
identical automaton states, refresh_tallies, single feedback calls,
update_clause and train_epoch_parallel(workers=1) in sync-mirror mode.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_io import EPOCH_CASES, load, manifest

pytestmark = pytest.mark.gpu

tm_mod = pytest.importorskip("paper_2009_04861_b200")
import paper_2009_04861_b200 as T  # noqa: E402


def _cfg(man, n=None):
    return T.TMConfig(clauses=n or man["n"], margin=man.get("margin", 15), specificity=man.get("s", 3.0),
                      state_depth=man["N"], boost_true_positive=bool(man.get("boost", 0)),
                      seed=man.get("seed", 42))


@pytest.mark.parametrize("o", [1, 2, 12, 31, 32, 33, 63, 64, 65, 100, 784])
def test_pool_literals_match_reference_packing(o):
    bits = load("pack", f"bits_o{o}.npy")
    pool = T.ExamplePool(o, bits, np.array([0, 1, 0], np.int32), 2)
    assert np.array_equal(pool.all_literals(), load("pack", f"lits_o{o}.npy"))


def test_pool_validation_errors():
    with pytest.raises(ValueError, match="0/1"):
        T.ExamplePool(3, np.array([[0, 2, 1]], np.uint8), np.array([0], np.int32), 2)
    with pytest.raises(ValueError, match="label"):
        T.ExamplePool(3, np.array([[0, 1, 1]], np.uint8), np.array([5], np.int32), 2)
    with pytest.raises(ValueError, match="empty"):
        T.ExamplePool(3, np.zeros((0, 3), np.uint8), np.zeros(0, np.int32), 2)


def test_counter_roundtrip_and_masks():
    for case in manifest("feedback"):
        k = case["idx"]
        before = load("feedback", f"case{k}_before.npy")
        tm = T.MultiClassTM(T.TMConfig(clauses=2, state_depth=case["N"]), case["o"], 1)
        tm.banks[0].set_counters(before)
        assert np.array_equal(tm.banks[0].counters(), before)
        ref = O.Machine(case["o"], 1, 2, case["N"])
        ref.set_counters(before[None])
        assert np.array_equal(tm.banks[0].include_masks(), ref.masks[0])
        assert np.array_equal(tm.banks[0].include_counts(), ref.counts[0])


def test_feedback_golden_cases():
    for case in manifest("feedback"):
        k = case["idx"]
        x = load("feedback", f"case{k}_x.npy")
        before = load("feedback", f"case{k}_before.npy")
        after = load("feedback", f"case{k}_after.npy")
        tm = T.MultiClassTM(T.TMConfig(clauses=2, state_depth=case["N"]), case["o"], 1)
        tm.banks[0].set_counters(before)
        lits = O.pack_literals(x)[0]
        r = T.Rng(case["rng_seed"], case["rng_stream"])
        if case["type"] == 1:
            T.type_i_feedback(tm.banks[0], 1, lits, case["s"], bool(case["boost"]), r)
        else:
            T.type_ii_feedback(tm.banks[0], 1, lits)
        assert np.array_equal(tm.banks[0].counters(), after), f"feedback case {k}"
        if case["type"] == 1:
            assert r.next() == int(case["next_draw"]), f"draw count, case {k}"


def _set_state(d, tag, tm, pool, m, q):
    counters = load(*d, f"{tag}_counters.npy")
    prev = load(*d, f"{tag}_prev.npy")
    tm.bind_examples(q)
    for c in range(m):
        tm.banks[c].set_counters(counters[c])
        tm.banks[c].set_prev_outputs(prev[c])
    pool.set_tallies(load(*d, f"{tag}_tallies.npy"))


def _check_state(d, tag, tm, pool, m):
    for c in range(m):
        b = tm.banks[c]
        assert np.array_equal(b.counters(), load(*d, f"{tag}_counters.npy")[c]), f"{tag} counters bank {c}"
        assert np.array_equal(b.include_masks(), load(*d, f"{tag}_masks.npy")[c]), f"{tag} masks bank {c}"
        assert np.array_equal(b.include_counts(), load(*d, f"{tag}_counts.npy")[c]), f"{tag} counts bank {c}"
        assert np.array_equal(b.prev_outputs(), load(*d, f"{tag}_prev.npy")[c]), f"{tag} prev bank {c}"
    assert np.array_equal(pool.tallies(), load(*d, f"{tag}_tallies.npy")), f"{tag} tallies"


def test_update_clause_golden_cases():
    for case in manifest("update_clause"):
        k = case["idx"]
        d = ("update_clause",)
        bits, labels = load(*d, f"case{k}_bits.npy"), load(*d, f"case{k}_labels.npy")
        order = load(*d, f"case{k}_order.npy")
        pool = T.ExamplePool(case["o"], bits, labels, case["m"])
        tm = T.MultiClassTM(T.TMConfig(clauses=case["n"], state_depth=case["N"]), case["o"], case["m"])
        _set_state(d, f"case{k}_in", tm, pool, case["m"], case["q"])
        r = T.Rng(case["rng_seed"], case["rng_stream"])
        ev = T.update_clause(tm.banks[case["cls"]], case["j"], pool, case["cls"], order, case["offset"],
                             case["batch"], case["margin"], case["s"], bool(case["boost"]), r)
        assert ev == case["events"], f"case {k}"
        _check_state(d, f"case{k}_out", tm, pool, case["m"])
        assert r.next() == int(case["next_draw"])


@pytest.mark.parametrize("name", EPOCH_CASES)
def test_sync_mirror_epochs_bit_exact(name):
    """train_epoch_parallel(workers=1) replayed on the GPU == the reference."""
    d = ("epoch_par_w1", name)
    man = manifest(*d)
    pool = T.ExamplePool(man["o"], load(*d, "train_x.npy"), load(*d, "train_y.npy"), man["m"])
    tm = T.MultiClassTM(_cfg(man), man["o"], man["m"])
    for ep in man["epochs"]:
        e = ep["epoch"]
        rep = T.train_epoch_parallel(tm, pool, 1, e, mode=T.MODE_SYNC_MIRROR)
        assert rep.feedback_events == ep["feedback_events"], f"events epoch {e}"
        _check_state(d, f"epoch{e}", tm, pool, man["m"])
    test = T.ExamplePool(man["o"], load(*d, "test_x.npy"), load(*d, "test_y.npy"), man["m"])
    assert np.array_equal(T.class_sums(tm, test), load(*d, "test_sums.npy"))
    assert np.array_equal(T.predict_all(tm, test), load(*d, "test_pred.npy"))
    assert T.evaluate_accuracy(tm, test) == pytest.approx(man["test_accuracy"], abs=0)
    T.refresh_tallies(pool, tm)
    _check_state(d, "refreshed", tm, pool, man["m"])


def test_auto_mode_rule(monkeypatch):
    """TMG_MODE_AUTO, the mode of the drop-in train_epoch_parallel in Python
    and in the C++ facade: asynchronous for any worker count; the bit-exact
    one-worker replay only with TSETLIN_DETERMINISTIC=1."""
    name = EPOCH_CASES[0]
    d = ("epoch_par_w1", name)
    man = manifest(*d)
    ep = man["epochs"][0]

    def run():
        pool = T.ExamplePool(man["o"], load(*d, "train_x.npy"), load(*d, "train_y.npy"), man["m"])
        cfg = T.TMConfig(clauses=man["n"], margin=man["margin"], specificity=man["s"], state_depth=man["N"],
                         boost_true_positive=bool(man["boost"]), seed=man["seed"])
        tm = T.MultiClassTM(cfg, man["o"], man["m"])
        return T.train_epoch_parallel(tm, pool, 1, ep["epoch"]), tm

    monkeypatch.delenv("TSETLIN_DETERMINISTIC", raising=False)
    rep, _ = run()
    assert sum(rep.type_i_events) > 0  # only the asynchronous engine reports Type I counts
    monkeypatch.setenv("TSETLIN_DETERMINISTIC", "1")
    rep, tm = run()
    assert rep.feedback_events == ep["feedback_events"] and sum(rep.type_i_events) == 0
    counters = load(*d, f"epoch{ep['epoch']}_counters.npy")
    for c in range(man["m"]):
        assert np.array_equal(tm.banks[c].counters(), counters[c])


@pytest.mark.parametrize("name,o,m,n", [("mnist_rand", 784, 10, 50), ("single_bank", 30, 1, 8),
                                        ("dense_o64", 64, 3, 12)])
def test_inference_random_states(name, o, m, n):
    bits = load("inference", f"{name}_bits.npy")
    tm = T.MultiClassTM(T.TMConfig(clauses=n), o, m)
    counters = load("inference", f"{name}_counters.npy")
    for c in range(m):
        tm.banks[c].set_counters(counters[c])
    pool = T.ExamplePool(o, bits, np.zeros(bits.shape[0], np.int32), m)
    sums = load("inference", f"{name}_sums.npy")
    assert np.array_equal(T.class_sums(tm, pool), sums)
    assert np.array_equal(T.predict_all(tm, pool), load("inference", f"{name}_pred.npy"))
    lits = O.pack_literals(bits)
    assert np.array_equal(T.export_vote_sums(tm, lits), sums)
    assert np.array_equal(T.export_vote_sums(tm, lits[3]), sums[3])
    assert T.classify(tm, lits[5]) == load("inference", f"{name}_pred.npy")[5]
    T.refresh_tallies(pool, tm)
    assert np.array_equal(pool.tallies(), load("inference", f"{name}_tallies.npy"))
    prev = load("inference", f"{name}_prev.npy")
    for c in range(m):
        assert np.array_equal(tm.banks[c].prev_outputs(), prev[c])


def test_inference_vs_oracle_random_large():
    """Class sums at a bigger random shape (many words, ties, empty clauses)."""
    rng = np.random.default_rng(7)
    o, m, n, q = 300, 4, 64, 777
    bits = (rng.random((q, o)) < 0.5).astype(np.uint8)
    counters = np.where(rng.random((m, n, 2 * o)) < 0.01, 129 + rng.integers(0, 128, (m, n, 2 * o)),
                        1 + rng.integers(0, 128, (m, n, 2 * o))).astype(np.uint16)
    counters[:, ::7, :] = 128  # empty clauses
    tm = T.MultiClassTM(T.TMConfig(clauses=n), o, m)
    for c in range(m):
        tm.banks[c].set_counters(counters[c])
    ref = O.Machine(o, m, n, 128)
    ref.set_counters(counters)
    pool = T.ExamplePool(o, bits, rng.integers(0, m, q).astype(np.int32), m)
    lits = O.pack_literals(bits)
    assert np.array_equal(T.class_sums(tm, pool), ref.class_sums(lits))
    assert np.array_equal(T.predict_all(tm, pool), ref.predict(lits))


def test_errors_follow_reference():
    tm = T.MultiClassTM(T.TMConfig(clauses=4), 12, 2)
    pool = T.ExamplePool(13, np.zeros((4, 13), np.uint8), np.zeros(4, np.int32), 2)
    with pytest.raises(ValueError, match="feature count mismatch"):
        T.train_epoch_parallel(tm, pool, 1, 0)
    pool2 = T.ExamplePool(12, np.zeros((4, 12), np.uint8), np.zeros(4, np.int32), 2)
    with pytest.raises(ValueError, match="workers"):
        T.train_epoch_parallel(tm, pool2, 0, 0)
    with pytest.raises(ValueError, match="batch"):
        T.update_clause(tm.banks[0], 0, pool2, 0, None, 0, 0, 15, 3.0, False, T.Rng(1))
    with pytest.raises(ValueError, match="order length"):
        T.update_clause(tm.banks[0], 0, pool2, 0, [0, 1], 0, 1, 15, 3.0, False, T.Rng(1))
    with pytest.raises(IndexError):
        tm.banks[0].set_counters  # accessor exists
        T.update_clause(tm.banks[1], 9, pool2, 1, None, 0, 1, 15, 3.0, False, T.Rng(1))


def test_update_clause_rejects_order_entries_out_of_range():
    """record_output_and_tally's bounds check (pool.cpp:95-98) -> out_of_range,
    raised before anything is written on the device."""
    tm = T.MultiClassTM(T.TMConfig(clauses=4), 12, 2)
    pool = T.ExamplePool(12, np.ones((4, 12), np.uint8), np.zeros(4, np.int32), 2)
    before = tm.banks[0].counters()
    for bad in ([0, 1, 2, 4], [0, -1, 2, 3]):
        with pytest.raises(IndexError, match="out of range"):
            T.update_clause(tm.banks[0], 0, pool, 0, bad, 0, 4, 15, 3.0, False, T.Rng(1))
    assert np.array_equal(tm.banks[0].counters(), before)
    assert not pool.tallies().any()


def test_update_clause_rebinds_only_its_bank():
    """update_clause rebinds the bank it updates (trainer.cpp:107); the other
    banks keep their bound count and previous outputs (core.cpp:117-126)."""
    tm = T.MultiClassTM(T.TMConfig(clauses=4, margin=15, specificity=3.0), 12, 2)
    small = T.ExamplePool(12, np.ones((10, 12), np.uint8), np.zeros(10, np.int32), 2)
    T.train_epoch_parallel(tm, small, 1, 0, mode=T.MODE_SYNC_MIRROR)
    prev0 = tm.banks[0].prev_outputs()
    assert tm.banks[0].bound_examples() == 10 and tm.banks[1].bound_examples() == 10
    big = T.ExamplePool(12, np.ones((100, 12), np.uint8), np.ones(100, np.int32), 2)
    T.update_clause(tm.banks[1], 1, big, 1, None, 0, 5, 15, 3.0, False, T.Rng(3))
    assert tm.banks[0].bound_examples() == 10 and tm.banks[1].bound_examples() == 100
    assert np.array_equal(tm.banks[0].prev_outputs(), prev0)
    assert tm.banks[1].prev_outputs().shape == (4, 2)
    assert tm.info().bound_examples == -1
    tm.banks[0].bind_examples(100)  # per bank again
    assert tm.banks[0].bound_examples() == 100 and not tm.banks[0].prev_outputs().any()
    assert tm.info().bound_examples == 100


@pytest.mark.parametrize("kind,q,n", [("mnist", 60, 200), ("imdb", 12, 60), ("xor", 300, 20), ("fmnist", 20, 100)])
def test_sequential_parallel_replay_matches_serial(kind, q, n, monkeypatch):
    """train_epoch_sequential's parallel replay (gate scan with xoshiro
    jump-ahead over the Type I draws, then every gated clause applied by its
    own warp from its recorded generator state; sequential.cu) leaves exactly
    the serial replay's automata, tallies and events — which
    test_gpu_dropin.py pins to the reference's goldens."""
    from paper_2009_04861_b200 import synth
    d = synth.make(kind, q, 4, 7)
    got = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("TMG_SEQ_SERIAL", mode)
        tm = T.MultiClassTM(T.TMConfig(clauses=n, margin=20, specificity=5.0, boost_true_positive=True, seed=3),
                            d.features, d.classes)
        pool = T.ExamplePool(d.features, d.train_x, d.train_y, d.classes)
        ev = [T.train_epoch_sequential(tm, pool, e).feedback_events for e in range(2)]
        got[mode] = (np.stack([tm.banks[c].counters() for c in range(d.classes)]), ev)
    assert got["0"][1] == got["1"][1]
    assert np.array_equal(got["0"][0], got["1"][0])


@pytest.mark.parametrize("kind,q,n", [("mnist", 40, 40), ("imdb", 6, 10)])
def test_w1_replay_jump_draws_match_serial(kind, q, n, monkeypatch):
    """train_epoch_parallel(workers=1)'s replay draws a Type I step's 2o
    uniforms by warp-cooperative jump-ahead when 2o >= 256 (train.cu
    draw_type_i_bits); it must leave exactly the automata, tallies and
    events of the serial draws (TMG_SEQ_SERIAL=1)."""
    from paper_2009_04861_b200 import synth
    d = synth.make(kind, q, 4, 11)
    got = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("TMG_SEQ_SERIAL", mode)
        tm = T.MultiClassTM(T.TMConfig(clauses=n, margin=10, specificity=4.0, seed=5), d.features, d.classes)
        pool = T.ExamplePool(d.features, d.train_x, d.train_y, d.classes)
        ev = [T.train_epoch_parallel(tm, pool, 1, e, mode=T.MODE_SYNC_MIRROR).feedback_events for e in range(2)]
        got[mode] = (np.stack([tm.banks[c].counters() for c in range(d.classes)]), pool.tallies(), ev)
    assert got["0"][2] == got["1"][2]
    assert np.array_equal(got["0"][0], got["1"][0])
    assert np.array_equal(got["0"][1], got["1"][1])
