"""Edge shapes of the reference's TMConfig / ExamplePool range
(core.cpp:48-74, pool.cpp:23-80) through the GPU engine: one feature, one
bank, one or two examples, the smallest and largest state depths (N = 1 ->
4 bit planes, N = 16383 -> 15), margin 1, s = 1, boost, widths straddling the
word and warp boundaries, and rows past every shared-memory capacity (the
reference has no width limit). Each runs the sync-mirror epoch against the oracle
(bit-exact) and asynchronous epochs under the tally invariant."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

T = pytest.importorskip("paper_2009_04861_b200")

CASES = [
    # name, o, m, n, N, T, s, boost, q
    ("one_feature", 1, 2, 2, 128, 1, 1.0, False, 7),
    ("one_example", 33, 2, 4, 128, 5, 3.0, False, 1),
    ("single_bank", 40, 1, 6, 100, 3, 2.0, True, 50),
    ("depth_1", 31, 3, 4, 1, 2, 1.5, False, 40),
    ("depth_16383", 64, 2, 4, 16383, 50, 10.0, False, 60),
    ("word_edges", 1025, 2, 2, 8, 4, 3.9, True, 30),
    ("many_classes", 20, 37, 2, 128, 3, 4.0, False, 200),
    # runtime-width rows: replay kernel with planes in place (> 16 384 features),
    # direct evaluation (> ~26k), async planes in HBM (> 107 520 at 8 planes,
    # > 57 344 at 15)
    ("wide_20k", 20000, 2, 2, 128, 6, 3.0, True, 48),
    ("wide_40k", 40000, 3, 2, 100, 4, 5.0, False, 40),
    ("wide_110k_inplace", 110000, 2, 2, 128, 5, 3.0, False, 33),
    ("wide_60k_deep_inplace", 60000, 2, 2, 9000, 8, 4.0, False, 20),
]


def _data(o, m, q, seed):
    rng = np.random.default_rng(seed)
    protos = rng.random((m, o)) < 0.4
    y = rng.integers(0, m, q).astype(np.int32)
    x = (protos[y] ^ (rng.random((q, o)) < 0.1)).astype(np.uint8)
    return x, y


@pytest.mark.parametrize("name,o,m,n,N,T_,s,boost,q", CASES)
def test_edge_shapes(name, o, m, n, N, T_, s, boost, q):
    x, y = _data(o, m, q, o + m + n)
    cfg = T.TMConfig(clauses=n, margin=T_, specificity=s, state_depth=N, boost_true_positive=boost, seed=5)
    # sync mirror: bit-exact vs the oracle's train_epoch_parallel(workers=1)
    tm = T.MultiClassTM(cfg, o, m)
    pool = T.ExamplePool(o, x, y, m)
    ref = O.Machine(o, m, n, N, q)
    rpool = O.Pool(x, y, m)
    for e in range(2):
        rep = T.train_epoch_parallel(tm, pool, 1, e, mode=T.MODE_SYNC_MIRROR)
        ev = O.train_epoch_parallel(ref, rpool, T_, s, boost, 5, 1, e)
        assert rep.feedback_events == [int(v) for v in ev], (name, e)
    got = np.stack([tm.banks[c].counters() for c in range(m)])
    assert np.array_equal(got, ref.counters), name
    assert np.array_equal(pool.tallies(), rpool.tallies), name
    # asynchronous epochs: invariant, counter range
    tm2 = T.MultiClassTM(cfg, o, m)
    pool2 = T.ExamplePool(o, x, y, m)
    for e in range(3):
        T.train_epoch_parallel(tm2, pool2, 1, e)
        tal = pool2.tallies()
        for c in range(m):
            b = np.unpackbits(tm2.banks[c].prev_outputs().view(np.uint8), axis=1, bitorder="little")[:, :q]
            b = b.astype(np.int64)
            assert np.array_equal(tal[:, c], b[0::2].sum(0) - b[1::2].sum(0)), (name, e, c)
    cs = np.stack([tm2.banks[c].counters() for c in range(m)])
    assert cs.min() >= 1 and cs.max() <= 2 * N
    # inference on the async state vs the oracle
    ref.set_counters(cs)
    lits = O.pack_literals(x)
    assert np.array_equal(T.class_sums(tm2, pool2), ref.class_sums(lits))
    assert np.array_equal(T.predict_all(tm2, pool2), ref.predict(lits))
