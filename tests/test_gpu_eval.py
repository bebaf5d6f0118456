"""Edge cases of the example-sliced class-sum kernel (csrc/eval.cu
eval_bits_kernel) against numpy restatements of vote_sum / refresh_tallies
(proj/src/pool.cpp:82-124, core.hpp:208-219): long and empty literal lists,
clause counts past one CTA's counter range (2040), example counts at the
32-bit word and 1024-example block edges, the train-mode previous-output
bitmaps."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

T = pytest.importorskip("paper_2009_04861_b200")


def _sums(counters, bits, N, train):
    """[q][m] class sums: counters [m][n][2o] (1..2N), bits [q][o] 0/1."""
    lit = np.concatenate([bits, 1 - bits], axis=1).astype(np.float64)
    out = np.zeros((bits.shape[0], counters.shape[0]), np.int64)
    outs = []
    for c in range(counters.shape[0]):
        inc = (counters[c] > N).astype(np.float64)
        fire = (inc @ (1.0 - lit).T) == 0  # [n][q]
        empty = inc.sum(axis=1) == 0
        fire[empty, :] = train  # core.hpp:211-213: empty clause -> Train 1 / Predict 0
        sign = np.where(np.arange(inc.shape[0]) % 2 == 0, 1, -1)
        out[:, c] = (fire * sign[:, None]).sum(axis=0)
        outs.append(fire)
    return out, outs


@pytest.mark.parametrize("q", [1, 33, 1025, 2500])
def test_long_lists_empty_clauses_and_chunks(q):
    rng = np.random.default_rng(q)
    o, m, n, N = 300, 3, 4100, 128  # n > 2040: several CTA chunks per class
    counters = np.full((m, n, 2 * o), N, np.uint16)
    dens = rng.choice([0.0, 0.002, 0.02, 0.3], size=(m, n))  # empty, sparse, medium, long lists
    for c in range(m):
        hit = rng.random((n, 2 * o)) < dens[c][:, None]
        counters[c][hit] = N + 1 + rng.integers(0, N, hit.sum())
    bits = (rng.random((q, o)) < 0.5).astype(np.uint8)
    tm = T.MultiClassTM(T.TMConfig(clauses=n), o, m)
    for c in range(m):
        tm.banks[c].set_counters(counters[c])
    pool = T.ExamplePool(o, bits, np.zeros(q, np.int32), m)
    want, _ = _sums(counters, bits.astype(np.int64), N, train=False)
    assert np.array_equal(T.class_sums(tm, pool), want)
    lits = pool.all_literals()
    assert np.array_equal(T.export_vote_sums(tm, lits), want)
    want_t, fires = _sums(counters, bits.astype(np.int64), N, train=True)
    assert np.array_equal(T.class_sums(tm, pool, T.TRAIN), want_t)
    T.refresh_tallies(pool, tm)  # also rewrites every previous-output bitmap
    assert np.array_equal(pool.tallies(), want_t)
    for c in range(m):
        prev = tm.banks[c].prev_outputs()
        got = np.unpackbits(prev.view(np.uint8), axis=1, bitorder="little")[:, :q].astype(bool)
        assert np.array_equal(got, fires[c])
        tail = np.unpackbits(prev.view(np.uint8), axis=1, bitorder="little")[:, q:]
        assert not tail.any()  # bits past q stay zero


def test_sum_range_past_one_cta():
    """Every positive clause empty (Train 1), every negative one falsified:
    each example's train-mode sum is n/2 = 3000, beyond the 12-bit counter
    planes of one CTA (|sum| <= 2040), so the chunking must split it."""
    o, n, N, q = 40, 6000, 128, 777
    counters = np.full((1, n, 2 * o), N, np.uint16)
    counters[0, 1::2, 0] = N + 1  # negative clauses include x_0 ...
    bits = np.zeros((q, o), np.uint8)  # ... which is 0 everywhere
    tm = T.MultiClassTM(T.TMConfig(clauses=n), o, 1)
    tm.banks[0].set_counters(counters[0])
    pool = T.ExamplePool(o, bits, np.zeros(q, np.int32), 1)
    assert (T.class_sums(tm, pool, T.TRAIN) == n // 2).all()
    assert (T.class_sums(tm, pool, T.PREDICT) == 0).all()  # empty positives vote 0 in predict mode
    assert (T.predict_all(tm, pool) == 1).all()  # one bank: sum >= 0 -> 1 (trainer.cpp:244-260)
