"""Host-side checks of the asynchronous sampler's alias table (no GPU): the
pattern law the engine samples for clause-output-0 Type I draws equals the
product law Bernoulli(P/2^32)^8 to within 2^-32 per pattern (so each
literal's marginal is within 2^-25 of P/2^32)."""
import numpy as np
import pytest

from oracle import oracle as O

T = pytest.importorskip("paper_2009_04861_b200")


@pytest.mark.parametrize("s", [1.0, 1.5, 2.0, 3.9, 10.0, 15.0, 25.0, 100.0, 1000.0])
def test_alias_table_law(s):
    from paper_2009_04861_b200.tsetlin import alias8_table
    thr = O.prob_threshold(1.0 / s)
    table = alias8_table(thr)
    law = O.alias8_law(table)
    p = thr / 2.0 ** 32
    k = np.array([bin(i).count("1") for i in range(256)])
    exact = p ** k * (1.0 - p) ** (8 - k)
    assert abs(law.sum() - 1.0) < 1e-12
    assert np.abs(law - exact).max() <= 2.0 ** -32 + 1e-15, np.abs(law - exact).max()
    # per-literal marginal: a sum of 128 pattern masses, each within 2^-32
    for b in range(8):
        marg = law[(np.arange(256) >> b) & 1 == 1].sum()
        assert abs(marg - p) <= 2.0 ** -25


def test_async_sampler_restatement_alias_rate():
    """Clause output 0 through the alias path of the restatement: pooled
    decrement rate 1/s on unsaturated automata."""
    from paper_2009_04861_b200.tsetlin import alias8_table
    o, N, s = 64, 128, 10.0
    table = alias8_table(O.prob_threshold(1.0 / s))
    counters = np.full(2 * o, 100, np.uint16)
    lits = O.pack_literals(np.zeros(o, np.uint8))[0]
    moved = 0
    trials = 400
    for i in range(trials):
        after = O.async_type_i(counters, lits, o, N, 0, s, False, 5, i, 1, 0, 1, alias8=table)
        assert ((after == counters) | (after == counters - 1)).all()
        moved += int((after != counters).sum())
    rate = moved / (trials * 2 * o)
    assert abs(rate - 0.1) < 0.006, rate
