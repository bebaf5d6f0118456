"""Asynchronous (Algorithm 1) training on the GPU: invariants, statistical
conformance and accuracy parity with the reference's parallel trainer."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_io import GOLDEN

pytestmark = pytest.mark.gpu

T = pytest.importorskip("paper_2009_04861_b200")
from paper_2009_04861_b200 import synth  # noqa: E402


def _bits_of(prev_words: np.ndarray, q: int) -> np.ndarray:
    """n x ceil(q/64) uint64 -> n x q {0,1} (bit i of word i//64)."""
    b = np.unpackbits(prev_words.view(np.uint8), axis=1, bitorder="little")
    return b[:, :q].astype(np.int64)


def _check_tally_invariant(tm, pool, m, q):
    """tally[i][c] == sum_j sign(j) * prev_bit[c][j][i] at quiescence
    (pool.cpp:71, core.cpp:123-125, pool.cpp:99-105)."""
    tallies = pool.tallies()
    for c in range(m):
        bits = _bits_of(tm.banks[c].prev_outputs(), q)
        expect = bits[0::2].sum(0) - bits[1::2].sum(0)
        assert np.array_equal(tallies[:, c], expect), f"class {c}"


def test_async_epoch_invariants_mnist_shape():
    d = synth.make("mnist", 3000, 500, 2009)
    cfg = T.TMConfig(clauses=200, margin=50, specificity=10.0, seed=3)
    tm = T.MultiClassTM(cfg, 784, 10)
    pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
    for e in range(2):
        rep = T.train_epoch_parallel(tm, pool, 1, e)
        assert rep.total_feedback_events() > 0
        assert 0 < sum(rep.type_i_events) < rep.total_feedback_events()
        _check_tally_invariant(tm, pool, 10, 3000)
    for c in range(10):
        cs = tm.banks[c].counters()
        assert cs.min() >= 1 and cs.max() <= 256
    # refresh: exact train-mode sums, and the same on the oracle for these states
    T.refresh_tallies(pool, tm)
    exact = T.class_sums(tm, pool, T.TRAIN)
    assert np.array_equal(pool.tallies(), exact)
    ref = O.Machine(784, 10, 200, 128)
    ref.set_counters(np.stack([tm.banks[c].counters() for c in range(10)]))
    rpool = O.Pool(d.train_x, d.train_y, 10)
    O.refresh_tallies(ref, rpool)
    assert np.array_equal(pool.tallies(), rpool.tallies)
    _check_tally_invariant(tm, pool, 10, 3000)
    # inference parity on the trained state
    test = T.ExamplePool(784, d.test_x, d.test_y, 10)
    lits = O.pack_literals(d.test_x)
    assert np.array_equal(T.class_sums(tm, test), ref.class_sums(lits))
    assert np.array_equal(T.predict_all(tm, test), ref.predict(lits))


@pytest.mark.parametrize("kind,q,clauses,T_,s_", [("fmnist", 800, 40, 100, 15.0), ("imdb", 600, 24, 100, 15.0)])
def test_async_epoch_invariants_wide_rows(kind, q, clauses, T_, s_):
    """Register kernel at 3 words per lane (FMNIST shape) and the shared-memory
    clause kernel (IMDb shape, 10 words per lane): tally invariant after every
    epoch, counters in range, exact refresh and inference vs the oracle."""
    d = synth.make(kind, q, 64, 7)
    tm = T.MultiClassTM(T.TMConfig(clauses=clauses, margin=T_, specificity=s_, seed=5), d.features, d.classes)
    pool = T.ExamplePool(d.features, d.train_x, d.train_y, d.classes)
    for e in range(2):
        rep = T.train_epoch_parallel(tm, pool, 1, e)
        assert 0 < sum(rep.type_i_events) < rep.total_feedback_events()
        _check_tally_invariant(tm, pool, d.classes, q)
    ref = O.Machine(d.features, d.classes, clauses, 128)
    ref.set_counters(np.stack([tm.banks[c].counters() for c in range(d.classes)]))
    assert ref.counters.min() >= 1 and ref.counters.max() <= 256
    T.refresh_tallies(pool, tm)
    rpool = O.Pool(d.train_x, d.train_y, d.classes)
    O.refresh_tallies(ref, rpool)
    assert np.array_equal(pool.tallies(), rpool.tallies)
    test = T.ExamplePool(d.features, d.test_x, d.test_y, d.classes)
    lits = O.pack_literals(d.test_x)
    assert np.array_equal(T.class_sums(tm, test), ref.class_sums(lits))


def test_two_clause_shards_one_gpu():
    """The multi-GPU window protocol (distributed.py) with two clause shards
    on one GPU and the all-reduce done by hand: after every epoch both tally
    replicas are equal and equal the signed sum of BOTH shards' clause
    outputs; sharded class sums (partial sums added) equal the oracle's on
    the combined state; accuracy is that of the unsharded machine."""
    import torch
    from paper_2009_04861_b200 import distributed as D
    d = synth.make("mnist", 3000, 1000, 2009)
    n, m, q = 200, 10, 3000
    cfg = T.TMConfig(clauses=n, margin=50, specificity=10.0, seed=4)
    engines = []
    for r in range(2):
        jb, je = D.shard_range(n, r, 2)
        tm = T.MultiClassTM(cfg, 784, m, clause_range=(jb, je))
        pool = T.ExamplePool(784, d.train_x, d.train_y, m)
        engines.append(D.GpuShardEngine(tm, pool))
    for e in range(2):
        for eng in engines:
            eng.begin(e)
        for t0, t1 in D.window_bounds(q, 8):
            for eng in engines:
                eng.window(e, t0, t1)
            torch.cuda.synchronize()
            reduced = engines[0].delta().clone() + engines[1].delta().clone()
            for eng in engines:
                eng.apply(reduced)
            torch.cuda.synchronize()
        t0_, t1_ = engines[0].pool.tallies(), engines[1].pool.tallies()
        assert np.array_equal(t0_, t1_)
        for c in range(m):
            bits = np.concatenate([_bits_of(eng.tm.banks[c].prev_outputs(), q) for eng in engines])
            expect = bits[0::2].sum(0) - bits[1::2].sum(0)
            assert np.array_equal(t0_[:, c], expect), (e, c)
    test = T.ExamplePool(784, d.test_x, d.test_y, m)
    sums = sum(T.class_sums(eng.tm, test) for eng in engines)
    ref = O.Machine(784, m, n, 128)
    full = np.concatenate([np.stack([eng.tm.banks[c].counters() for c in range(m)]) for eng in engines], axis=1)
    ref.set_counters(full)
    lits = O.pack_literals(d.test_x)
    assert np.array_equal(sums, ref.class_sums(lits))
    acc_sharded = float((sums.argmax(1) == d.test_y).mean())
    single = T.MultiClassTM(cfg, 784, m)
    spool = T.ExamplePool(784, d.train_x, d.train_y, m)
    for e in range(2):
        T.train_epoch_parallel(single, spool, 1, e)
    acc_single = T.evaluate_accuracy(single, test)
    assert acc_sharded > acc_single - 0.03, (acc_sharded, acc_single)


@pytest.mark.parametrize("o", [5000, 15000, 20000])
def test_async_epoch_invariants_very_wide(o):
    """Shared-memory clause kernels at 6 and 16 words per lane and the
    runtime-width instantiation (20 000 features, 20 words per lane) on random
    prototype data: tally invariant, counter range, exact refresh."""
    rng = np.random.default_rng(o)
    m, q, n = 3, 256, 8
    protos = rng.random((m, o)) < 0.3
    y = rng.integers(0, m, q).astype(np.int32)
    x = (protos[y] ^ (rng.random((q, o)) < 0.1)).astype(np.uint8)
    tm = T.MultiClassTM(T.TMConfig(clauses=n, margin=10, specificity=5.0, seed=2), o, m)
    pool = T.ExamplePool(o, x, y, m)
    for e in range(2):
        rep = T.train_epoch_parallel(tm, pool, 1, e)
        assert rep.total_feedback_events() > 0
        _check_tally_invariant(tm, pool, m, q)
    cs = np.stack([tm.banks[c].counters() for c in range(m)])
    assert cs.min() >= 1 and cs.max() <= 256
    T.refresh_tallies(pool, tm)
    ref = O.Machine(o, m, n, 128)
    ref.set_counters(cs)
    rpool = O.Pool(x, y, m)
    O.refresh_tallies(ref, rpool)
    assert np.array_equal(pool.tallies(), rpool.tallies)


def test_async_gate_zero_at_margin():
    """SPEC acceptance 2 on the asynchronous kernel: a step whose clamped
    class sum already sits at the margin (v = T for the label class, v = -T
    for the others) is never fed back (e = 0, feedback.cpp:24-28). Tallies
    preset far beyond +-T stay clamped there whatever the clauses do, so the
    whole epoch must report zero feedback events."""
    d = synth.make("mnist", 1000, 16, 2009)
    T_ = 20
    tm = T.MultiClassTM(T.TMConfig(clauses=100, margin=T_, specificity=10.0, seed=8), 784, 10)
    pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
    tal = np.full((1000, 10), -100000, np.int32)
    tal[np.arange(1000), d.train_y] = 100000
    pool.set_tallies(tal)
    rep = T.train_epoch_parallel(tm, pool, 1, 0)
    assert rep.total_feedback_events() == 0
    # one notch inside the margin for the label class only: every example of
    # class c gates its class-c clauses with probability 1/(2T) > 0
    tal[np.arange(1000), d.train_y] = T_ - 1
    pool.set_tallies(tal)
    tm.reset()
    rep = T.train_epoch_parallel(tm, pool, 1, 1)
    assert 0 < rep.total_feedback_events() < 1000 * 100 // 4


def test_async_contended_tallies_lose_no_update():
    """SPEC acceptance 6 (lost-update freedom) at GPU scale: 4 examples, 2
    classes x 2000 clauses, so every tally takes thousands of concurrent
    atomic adds per epoch; the tally invariant must hold exactly."""
    rng = np.random.default_rng(6)
    x = (rng.random((4, 64)) < 0.5).astype(np.uint8)
    y = np.array([0, 1, 0, 1], np.int32)
    tm = T.MultiClassTM(T.TMConfig(clauses=2000, margin=1000, specificity=3.0, seed=6), 64, 2)
    pool = T.ExamplePool(64, x, y, 2)
    for e in range(3):
        rep = T.train_epoch_parallel(tm, pool, 1, e)
        assert rep.total_feedback_events() > 4000
        _check_tally_invariant(tm, pool, 2, 4)


def test_async_window_accounting():
    """Windows of a pass compose to the full pass (multi-GPU building block)."""
    d = synth.make("xor", 1000, 10, 5, 0.1)
    cfg = T.TMConfig(clauses=20, margin=15, specificity=3.9, seed=9)
    tm = T.MultiClassTM(cfg, 12, 2)
    pool = T.ExamplePool(12, d.train_x, d.train_y, 2)
    from paper_2009_04861_b200 import distributed as D
    ev = D.train_epoch_windows(D.GpuShardEngine(tm, pool), 0, windows=7, allreduce=None)
    assert sum(ev) > 0
    _check_tally_invariant(tm, pool, 2, 1000)


@pytest.mark.parametrize("o,N,s,boost,out", [(12, 128, 3.9, False, 0), (12, 128, 3.9, False, 1),
                                             (12, 128, 4.0, True, 1), (784, 128, 10.0, False, 0),
                                             (784, 128, 10.0, False, 1), (40, 5, 2.0, False, 1),
                                             (12, 128, 1.5, False, 0), (12, 128, 1.5, False, 1),
                                             (12, 128, 15.0, False, 0), (12, 128, 15.0, True, 1)])
def test_type_i_table1_conformance(o, N, s, boost, out):
    """SPEC acceptance 1: Table 1 transition frequencies of the
    asynchronous Philox/bit-serial sampler within +-0.02 over 1e5 draws, at
    the criterion's s = 1.5, 4, 15 and the configs' 3.9 and 10."""
    from paper_2009_04861_b200.tsetlin import feedback_rates
    rng = np.random.default_rng(o + N)
    x = (rng.random(o) < 0.5).astype(np.uint8)
    lits = O.pack_literals(x)[0]
    L = 2 * o
    litv = np.concatenate([x, 1 - x]).astype(bool)
    # counters away from the saturation ends; includes only on true literals
    # when the clause must fire (out = 1), a few includes otherwise.
    counters = rng.integers(2, 2 * N, size=(2, L)).astype(np.uint16)
    counters[counters == N + 1] = N + 2 if N + 2 < 2 * N else N
    inc_lit = rng.random(L) < 0.1
    if out:
        inc_lit &= litv
    counters[1] = np.where(inc_lit, np.maximum(counters[1], N + 1), np.minimum(counters[1], N))
    tm = T.MultiClassTM(T.TMConfig(clauses=2, state_depth=N, specificity=s, boost_true_positive=boost), o, 1)
    tm.banks[0].set_counters(counters)
    assert T.evaluate_clause(tm.banks[0], 1, lits, T.TRAIN) == out or not out
    trials = 100_000
    inc, dec = feedback_rates(tm.banks[0], 1, lits, out, trials)
    inc, dec = inc / trials, dec / trials
    c = counters[1].astype(int)
    at_hi, at_lo = c == 2 * N, c == 1
    included = c > N
    p_hi, p_lo = (s - 1) / s, 1 / s
    if out:
        exp_inc = np.where(litv, np.where(included & boost, 1.0, p_hi), np.where(included, p_lo, 0.0))
        exp_dec = np.where(litv, 0.0, np.where(included, 0.0, p_lo))
    else:
        exp_inc = np.zeros(L)
        exp_dec = np.full(L, p_lo)
    exp_inc[at_hi] = 0.0
    exp_dec[at_lo] = 0.0
    assert np.abs(inc - exp_inc).max() < 0.02, np.abs(inc - exp_inc).max()
    assert np.abs(dec - exp_dec).max() < 0.02, np.abs(dec - exp_dec).max()
    # pooled check at 1e5 * L draws: mean rate of the p_lo decrements
    sel = exp_dec > 0
    if sel.sum() > 20:
        assert abs(dec[sel].mean() - p_lo) < 0.003


@pytest.mark.parametrize("o,N,s,boost", [(784, 128, 10.0, False), (784, 128, 10.0, True), (784, 100, 10.0, False),
                                         (12, 128, 3.9, False), (40, 5, 2.0, True), (2352, 128, 15.0, False),
                                         (1500, 300, 7.5, False), (2000, 128, 1.0, False),
                                         # the packed last word slot at its edge: 16 valid words
                                         # (packed) and 17 (plain), ClausePk in csrc/clause.cuh
                                         (1536, 128, 10.0, False), (1537, 128, 10.0, True),
                                         (5000, 128, 15.0, False), (10000, 128, 15.0, True),
                                         (9000, 100, 25.0, False), (15000, 128, 10.0, False),
                                         (20000, 128, 10.0, False), (40000, 5, 3.0, True)])
def test_async_type_i_bit_exact(o, N, s, boost):
    """The asynchronous Type I draw (Philox counters (clause, example) under the
    epoch key; alias-table patterns, or the exact bit-serial sampler when
    p_high != 1 - p_low; saturating steps) reproduced counter-for-counter by
    its C restatement (oracle/tm_oracle_async.c), for both clause outputs, on
    near-saturated and mid-range automata, register-resident and
    shared-memory (wide-row) clause paths."""
    from paper_2009_04861_b200.tsetlin import alias8_table, type_i_async
    rng = np.random.default_rng(o * 7 + N)
    table = alias8_table(O.prob_threshold(1.0 / s))
    n, m = 4, 2
    tm = T.MultiClassTM(T.TMConfig(clauses=n, state_depth=N, specificity=s, boost_true_positive=boost, seed=77),
                        o, m)
    nw = tm.info().words_per_lane
    L = 2 * o
    for c in range(m):
        cs = rng.integers(1, 2 * N + 1, size=(n, L))
        ends = rng.random((n, L))
        cs[ends < 0.15] = 1
        cs[ends > 0.9] = 2 * N
        tm.banks[c].set_counters(cs.astype(np.uint16))
    for trial in range(12):
        c, j = int(rng.integers(m)), int(rng.integers(n))
        x = (rng.random(o) < 0.5).astype(np.uint8)
        lits = O.pack_literals(x)[0]
        out = int(trial % 2)
        example, epoch = int(rng.integers(0, 1 << 31)), int(rng.integers(0, 50))
        before = tm.banks[c].counters()
        g = c * n + j
        expect = O.async_type_i(before[j], lits, o, N, out, s, boost, g, example, 77, epoch, nw, alias8=table)
        type_i_async(tm.banks[c], j, lits, out, example, epoch)
        after = tm.banks[c].counters()
        assert np.array_equal(after[j], expect), (trial, np.flatnonzero(after[j] != expect)[:10])
        others = [k for k in range(n) if k != j]
        assert np.array_equal(after[others], before[others])
        assert (after[j] != before[j]).any() or s == 1.0


def _ref_acc():
    path = os.path.join(GOLDEN, "accuracy_ref.json")
    return json.load(open(path)) if os.path.exists(path) else {}


@pytest.mark.parametrize("case,tol", [("xor_noise10", 0.005), ("xor_noise40", 0.01)])
def test_async_accuracy_parity_xor(case, tol):
    """Noisy XOR (SPEC acceptance 3/4): mean over 20 GPU seeds vs the
    reference's 5-seed mean; 40 % noise uses the spec's 2 pt parity band
    (SPEC.md:533). At 40 % noise the accuracy depends on the asynchronous
    schedule itself: the reference measures 0.953 with one worker and
    0.982-0.988 with eight."""
    ref = _ref_acc().get(case)
    if ref is None:
        pytest.skip("accuracy_ref.json lacks " + case)
    cfgd = ref["config"]
    accs = []
    for seed in range(1, 21):
        d = synth.make("xor", cfgd["q"], cfgd["qtest"], cfgd["data_seed"], cfgd["noise"])
        tm = T.MultiClassTM(T.TMConfig(clauses=cfgd["clauses"], margin=cfgd["T"], specificity=cfgd["s"],
                                       seed=seed), 12, 2)
        pool = T.ExamplePool(12, d.train_x, d.train_y, 2)
        test = T.ExamplePool(12, d.test_x, d.test_y, 2)
        for e in range(cfgd["epochs"]):
            T.train_epoch_parallel(tm, pool, 1, e)
        accs.append(T.evaluate_accuracy(tm, test))
    gpu, cpu = float(np.mean(accs)), ref["mean_final"]
    w1 = _ref_acc().get(case + "_w1")
    print(f"{case}: gpu mean {gpu:.4f} vs reference mean {cpu:.4f} (W={ref['workers']})"
          + (f", {w1['mean_final']:.4f} (W=1)" if w1 else "") + f" (per-seed {accs})")
    # The reference's own asynchronous schedules span [W=1 mean, W=8 mean];
    # the fully concurrent GPU schedule must land inside that band (+- tol).
    lo = min(cpu, w1["mean_final"]) if w1 else cpu
    hi = max(cpu, w1["mean_final"]) if w1 else cpu
    assert lo - tol <= gpu <= hi + tol


def _two_sided(gpu_accs, ref):
    """|GPU mean - reference mean| <= max(0.5 pt, 2 standard errors of the
    difference of the two seed means): on the small training prefixes one
    seed's accuracy moves by several points (IMDb q = 4000: 0.83-0.95 over
    the reference's own 5 seeds), so 0.5 pt alone is below what 5 seeds
    resolve. Returns (delta, tolerance)."""
    r = np.array([v[-1] for v in ref["per_seed"].values()])
    g = np.asarray(gpu_accs)
    se = np.sqrt(g.var(ddof=1) / len(g) + r.var(ddof=1) / len(r))
    return float(g.mean() - r.mean()), max(0.005, 2.0 * float(se))


def accuracy_parity(case, gpu_accs):
    """The parity rule for asynchronous training (BASELINE.json: <= 0.5 pt,
    mean over 5 seeds): the GPU's seed mean must lie within the reference's
    own spread of asynchronous schedules — its seed means over the worker
    counts measured (`case` = all host threads, `case`_w1/_w2/_w4 when
    accuracy_ref.json has them) — widened on both sides by
    max(0.5 pt, 2 standard errors). Returns (ok, message)."""
    acc = _ref_acc()
    ref = acc[case]
    delta, tol = _two_sided(gpu_accs, ref)
    means = {k: acc[k]["mean_final"] for k in (case, case + "_w1", case + "_w2", case + "_w4") if k in acc}
    lo, hi = min(means.values()), max(means.values())
    gpu = float(np.mean(gpu_accs))
    msg = (f"{case}: gpu mean {gpu:.4f}, reference means over W {means}, band [{lo - tol:.4f}, {hi + tol:.4f}] "
           f"(tolerance {tol:.4f}; per-seed {list(np.round(gpu_accs, 4))})")
    return lo - tol <= gpu <= hi + tol, msg


@pytest.mark.parametrize("case,kind", [("fmnist_q1000", "fmnist"), ("imdb_q4000", "imdb"),
                                       ("fmnist_q6000", "fmnist"), ("imdb_q12000", "imdb")])
def test_async_accuracy_parity_wide(case, kind):
    """BASELINE.json configs[2]/[3] shapes (FMNIST 2352 bits x 8000 clauses,
    IMDb 10 000 bits x 10 000 clauses, the shared-memory clause kernel) vs the
    reference's parallel trainer on the same training prefix, 5 seeds."""
    ref = _ref_acc().get(case)
    if ref is None:
        pytest.skip("accuracy_ref.json lacks " + case)
    cfgd = ref["config"]
    d = synth.make(kind, cfgd["q"], cfgd["qtest"], cfgd["data_seed"])
    accs = []
    for seed in range(1, 11):
        tm = T.MultiClassTM(T.TMConfig(clauses=cfgd["clauses"], margin=cfgd["T"], specificity=cfgd["s"],
                                       seed=seed), d.features, d.classes)
        pool = T.ExamplePool(d.features, d.train_x, d.train_y, d.classes)
        test = T.ExamplePool(d.features, d.test_x, d.test_y, d.classes)
        for e in range(cfgd["epochs"]):
            T.train_epoch_parallel(tm, pool, 1, e)
        accs.append(T.evaluate_accuracy(tm, test))
    ok, msg = accuracy_parity(case, accs)
    print(msg)
    assert ok, msg


def test_async_accuracy_parity_mnist():
    ref = _ref_acc().get("mnist_q6000")
    if ref is None:
        pytest.skip("accuracy_ref.json lacks mnist_q6000")
    cfgd = ref["config"]
    d = synth.make("mnist", cfgd["q"], cfgd["qtest"], cfgd["data_seed"])
    accs = []
    for seed in range(1, 6):
        tm = T.MultiClassTM(T.TMConfig(clauses=cfgd["clauses"], margin=cfgd["T"], specificity=cfgd["s"],
                                       seed=seed), 784, 10)
        pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
        test = T.ExamplePool(784, d.test_x, d.test_y, 10)
        for e in range(cfgd["epochs"]):
            T.train_epoch_parallel(tm, pool, 1, e)
        accs.append(T.evaluate_accuracy(tm, test))
    ok, msg = accuracy_parity("mnist_q6000", accs)
    print(msg)
    assert ok, msg


def _band(case):
    """The reference's own asynchronous-schedule spread at a configuration:
    [min, max] of its mean final accuracy over the worker counts measured
    (W = hardware threads, and the _w1/_w2/_w4 variants when present)."""
    acc = _ref_acc()
    means = [acc[k]["mean_final"] for k in (case, case + "_w1", case + "_w2", case + "_w4") if k in acc]
    return min(means), max(means), {k: acc[k]["mean_final"] for k in (case, case + "_w1", case + "_w2", case + "_w4")
                                    if k in acc}


def test_async_accuracy_parity_mnist_full():
    """The configuration bench.py times (BASELINE.json configs[1]): q = 60 000
    training rows, 10 000 test rows, 2000 clauses/class, T = 50, s = 10, three
    epochs, five seeds. Two-sided after EVERY epoch: the GPU's 5-seed mean
    lies within 0.5 pt of the band the reference's own asynchronous schedules
    span at that epoch — its seed means over the worker counts measured (all
    host threads, W = 4, W = 2, W = 1; tests/golden/accuracy_ref.json,
    gen_accuracy_ref.py). The reference itself moves by 3.5 pt at epoch 0
    between W = 8 (0.906) and W = 1 (0.941)."""
    acc = _ref_acc()
    ref = acc.get("mnist_q60000")
    if ref is None:
        pytest.skip("accuracy_ref.json lacks mnist_q60000")
    cfgd = ref["config"]
    d = synth.make("mnist", cfgd["q"], cfgd["qtest"], cfgd["data_seed"])
    per_epoch = np.zeros((5, cfgd["epochs"]))
    pool = T.ExamplePool(784, d.train_x, d.train_y, 10)
    test = T.ExamplePool(784, d.test_x, d.test_y, 10)
    for k, seed in enumerate(range(1, 6)):
        tm = T.MultiClassTM(T.TMConfig(clauses=cfgd["clauses"], margin=cfgd["T"], specificity=cfgd["s"],
                                       seed=seed), 784, 10)
        pool.reset_tallies()
        for e in range(cfgd["epochs"]):
            T.train_epoch_parallel(tm, pool, 8, e)
            per_epoch[k, e] = T.evaluate_accuracy(tm, test)
    gpu = per_epoch.mean(axis=0)
    curves = {k: np.mean([v for v in acc[k]["per_seed"].values()], axis=0)
              for k in ("mnist_q60000", "mnist_q60000_w4", "mnist_q60000_w2", "mnist_q60000_w1") if k in acc}
    lo = np.min(list(curves.values()), axis=0)
    hi = np.max(list(curves.values()), axis=0)
    print(f"mnist_q60000 per-epoch gpu {np.round(gpu, 4)}; reference per W "
          f"{ {k: np.round(v, 4).tolist() for k, v in curves.items()} }; gpu per seed {per_epoch[:, -1]}")
    for e in range(cfgd["epochs"]):
        assert lo[e] - 0.005 <= gpu[e] <= hi[e] + 0.005, (e, gpu, lo, hi)
