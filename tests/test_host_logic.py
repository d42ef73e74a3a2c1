"""Host-side logic that needs no GPU: validation, predicates, budgets, RNG,
meter, round driver — checked against the reference where it is present."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2103_01216_b200 import pred as P
from paper_2103_01216_b200 import runtime as R
from paper_2103_01216_b200.detres import LivelockError, RoundStats
from paper_2103_01216_b200.relaxed import decompose_driver, make_swap_sequence


def test_as_words_validation():
    R.as_words(np.zeros(3, dtype=np.uint64))
    for bad in (np.zeros(3, dtype=np.int64), np.zeros((2, 2), dtype=np.uint64),
                np.zeros(6, dtype=np.uint64)[::2], [1, 2, 3]):
        with pytest.raises(TypeError):
            R.as_words(bad)
    import torch

    with pytest.raises(TypeError):  # CPU tensors are not device words
        R.as_words(torch.zeros(3, dtype=torch.int64))
    with pytest.raises(TypeError):
        R.as_words(torch.zeros(3, dtype=torch.float32))


def test_pred_numpy_semantics_match_reference_lambdas():
    x = np.random.default_rng(1).integers(0, 1 << 64, size=10_000, dtype=np.uint64)
    W = np.uint64
    cases = [(P.even(), lambda b: (b & W(1)) == 0), (P.odd(), lambda b: (b & W(1)) == 1),
             (P.mod_eq(3, 0), lambda b: (b % W(3)) == 0), (P.lt(1 << 40), lambda b: b < W(1 << 40)),
             (P.eq(int(x[5])), lambda b: b == x[5]), (P.bit_set(7), lambda b: (b >> W(7)) & W(1) == 1),
             (~P.even(), lambda b: (b & W(1)) != 0), (P.always(), lambda b: np.ones(len(b), bool))]
    for p, f in cases:
        assert np.array_equal(p(x), f(x)), p


def test_plain_callable_rejected():
    with pytest.raises(TypeError):
        P.as_pred(lambda b: b > 1)


def test_epsilon_config():
    cfg = R.EpsilonConfig(0.5)
    assert cfg.prefix_words(10**6) == 20000
    assert cfg.prefix_words(1 << 30) == 21474836
    assert cfg.prefix_words(0) == 1
    assert R.EpsilonConfig(0.5, 1.0).prefix_words(8) == 8
    assert R.EpsilonConfig(0.5, 1e-12).prefix_words(65536) == 256
    with pytest.raises(ValueError):
        R.EpsilonConfig(1.0)
    with pytest.raises(ValueError):
        R.EpsilonConfig(0.5, 0.0)


def test_space_meter():
    m = R.SpaceMeter()
    rep = R.meter_scope(m, 10, lambda: (m.acquire(7), m.release(7)))
    assert rep.peak_words == 7 and not rep.exceeded and m.current_words == 0
    with pytest.raises(RuntimeError):
        m.release(1)


def test_decompose_driver():
    assert decompose_driver(100, 100, lambda h: h).rounds == 1
    st = decompose_driver(100, 10, lambda h: 10)
    assert st.rounds == 10 and st.committed_per_round == [10] * 10
    with pytest.raises(LivelockError):
        decompose_driver(5, 2, lambda h: 0)
    assert RoundStats(3, [1, 2, 3]).total_committed == 6


@pytest.mark.reference
def test_host_logic_vs_reference(ref):
    for n in (0, 1, 7, 10**5, 10**6, 1 << 30):
        for eps, f in ((0.5, 0.02), (0.3, 1e-12), (0.7, 1e-12), (0.5, 1.0)):
            assert R.EpsilonConfig(eps, f).prefix_words(n) == \
                ref.runtime.EpsilonConfig(eps, f).prefix_words(n)
    for seed in (0, 3, 177):
        assert np.array_equal(R.Rng(seed).words(0, 777), ref.runtime.Rng(seed).words(0, 777))
        assert R.Rng(seed).word(12) == ref.runtime.Rng(seed).word(12)
        assert R.Rng(seed).derive(5).seed == ref.runtime.Rng(seed).derive(5).seed
        assert np.array_equal(make_swap_sequence(1000, R.Rng(seed)),
                              ref.relaxed.make_swap_sequence(1000, ref.runtime.Rng(seed)))


def test_charges_reach_the_callers_pipal_meter(ref):
    """A pipal user measuring a drop-in call inside pipal.runtime.metered
    sees the GPU workspace words (runtime.py:194-253 of the reference)."""
    from paper_2103_01216_b200 import runtime as rt

    pm = ref.runtime.SpaceMeter()
    own = rt.SpaceMeter()
    with ref.runtime.metered(pm):
        ms = rt.charge(123)
        assert pm.current_words == 123
        rt.uncharge(123, ms)
        with rt.metered(own):
            ms = rt.charge(7)
            assert own.current_words == 7 and pm.current_words == 7
            rt.uncharge(7, ms)
    assert pm.current_words == 0 and pm.peak_words == 123 and own.peak_words == 7
    # no pipal meter active: only the drop-in's own meter is charged
    with rt.metered(own):
        ms = rt.charge(5)
        assert len(ms) == 1 and own.current_words == 5
        rt.uncharge(5, ms)
