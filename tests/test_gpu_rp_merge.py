"""GPU parity: random permutation (output AND round structure) and merge."""
from __future__ import annotations

import itertools

import numpy as np
import pytest

from conftest import golden, rand_words

pytestmark = pytest.mark.gpu

VARIANTS = ("naive", "flat", "oneres", "final")


def dev(a: np.ndarray):
    import torch

    return torch.from_numpy(a.view(np.int64).copy()).cuda()


def host(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


@pytest.fixture(scope="module")
def pip():
    import paper_2103_01216_b200 as pip

    return pip


def seq(orc, n, h):
    a = np.arange(n, dtype=np.uint64)
    orc.seq_knuth_shuffle(a, h)
    return a


# ----------------------------------------------------------------- RP

def test_rp_fig3_worked_example(pip, orc):
    h = np.array([0, 0, 1, 3, 1, 2, 3, 1], dtype=np.uint64)
    full = pip.EpsilonConfig(0.5, prefix_fraction=1.0)
    for v in VARIANTS:
        a = np.arange(8, dtype=np.uint64)
        tr = []
        pip.relaxed.random_permutation(a, h, variant=v, budget=full, trace=tr)
        assert sorted(tr[0].tolist()) == [5, 6, 7]
        assert a.tolist() == seq(orc, 8, h).tolist()


def test_rp_all_self_is_identity(pip):
    n = 64
    a = np.arange(n, dtype=np.uint64)
    st = pip.relaxed.random_permutation(a, np.arange(n, dtype=np.uint64))
    assert a.tolist() == list(range(n)) and st.rounds == 0


def test_rp_invalid(pip):
    with pytest.raises(ValueError):
        pip.relaxed.validate_swap_sequence(np.array([0, 2], dtype=np.uint64))
    with pytest.raises(ValueError):
        pip.relaxed.random_permutation(np.arange(2, dtype=np.uint64),
                                       np.array([0, 2], dtype=np.uint64))
    with pytest.raises(ValueError):
        pip.relaxed.random_permutation(np.arange(3, dtype=np.uint64),
                                       np.zeros(2, dtype=np.uint64))
    with pytest.raises(ValueError):
        pip.relaxed.random_permutation(np.arange(3, dtype=np.uint64),
                                       np.zeros(3, dtype=np.uint64), variant="bogus")


@pytest.mark.parametrize("variant", VARIANTS)
def test_rp_exhaustive_small(pip, orc, variant):
    full = pip.EpsilonConfig(0.5, prefix_fraction=1.0)
    for n in range(1, 6):
        for tail in itertools.product(*(range(i + 1) for i in range(1, n))):
            h = np.array((0,) + tail, dtype=np.uint64)
            a = np.arange(n, dtype=np.uint64)
            pip.relaxed.random_permutation(a, h, variant=variant, budget=full)
            assert np.array_equal(a, seq(orc, n, h)), (n, h.tolist())


def test_rp_golden_round_structure(pip):
    """rounds, committed_per_round, peak_table_load and trace equal the
    reference's (fixtures generated from pipal by tests/golden/make_golden.py)."""
    g = golden("rp")
    names = sorted({k.split("__")[0] for k in g.files})
    assert names
    for name in names:
        h = g[name + "__h"]
        n = len(h)
        eps, frac = (float(v) for v in g[name + "__budget"])
        variant = str(g[name + "__variant"][0])
        a = np.arange(n, dtype=np.uint64)
        tr = []
        st = pip.relaxed.random_permutation(dev(a) if n % 2 else a, h, variant,
                                            pip.EpsilonConfig(eps, frac), trace=tr)
        assert st.rounds == int(g[name + "__rounds"][0]), name
        assert st.committed_per_round == g[name + "__committed"].tolist(), name
        assert st.peak_table_load == float(g[name + "__peak"][0]), name
        assert np.array_equal(np.concatenate(tr) if tr else np.empty(0, np.uint64),
                              g[name + "__trace"]), name


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("n,seed,eps,frac", [(10_000, 177, 0.5, 0.02), (3000, 9, 0.5, 0.02),
                                             (20_000, 3, 0.7, 1e-12), (100_000, 55, 0.5, 0.02),
                                             (1_000_000, 1, 0.5, 0.02), (65_536, 7, 0.3, 1e-12)])
def test_rp_vs_oracle_rounds(pip, orc, variant, n, seed, eps, frac):
    rng = pip.Rng(seed)
    h = pip.relaxed.make_swap_sequence(n, rng)
    budget = pip.EpsilonConfig(eps, frac)
    a = dev(np.arange(n, dtype=np.uint64))
    st = pip.relaxed.random_permutation(a, dev(h), variant, budget)
    b = np.arange(n, dtype=np.uint64)
    ref = orc.ref_random_permutation(b, h, budget.prefix_words(n), variant, threads=8)
    assert np.array_equal(host(a), b)
    assert np.array_equal(b, seq(orc, n, h))
    assert st.rounds == ref["rounds"]
    assert st.committed_per_round == ref["committed_per_round"]
    assert st.peak_table_load == ref["peak_count"] / ref["capacity"]
    assert st.total_committed == int(np.count_nonzero(h != np.arange(n, dtype=np.uint64)))


def test_rp_adversarial_all_zero_targets(pip, orc):
    # every iterate targets 0: one commit per round (rounds == n - 1)
    n = 3000
    h = np.zeros(n, dtype=np.uint64)
    a = np.arange(n, dtype=np.uint64)
    st = pip.relaxed.random_permutation(a, h, budget=pip.EpsilonConfig(0.5, 0.05))
    assert np.array_equal(a, seq(orc, n, h))
    assert st.rounds == n - 1 and st.total_committed == n - 1


def test_rp_pcg64_input_config0(pip, orc):
    # BASELINE config 0: H[i] uniform in [0, i] from a PCG64 seed
    n = 1_000_000
    g = np.random.Generator(np.random.PCG64(1))
    h = g.integers(0, np.arange(1, n + 1, dtype=np.int64), dtype=np.int64).astype(np.uint64)
    a = dev(np.arange(n, dtype=np.uint64))
    pip.relaxed.random_permutation(a, dev(h))
    assert np.array_equal(host(a), seq(orc, n, h))


def test_rp_budget_metering(pip, orc):
    n = 100_000
    h = pip.relaxed.make_swap_sequence(n, pip.Rng(55))
    budget = pip.EpsilonConfig(0.5)
    b = budget.prefix_words(n)
    meter = pip.SpaceMeter()
    a = np.arange(n, dtype=np.uint64)
    rep = pip.meter_scope(meter, 8 * b,
                          lambda: pip.relaxed.random_permutation(a, h, budget=budget))
    assert rep.peak_words <= 8 * b, (rep.peak_words, 8 * b)
    assert meter.current_words == 0
    assert np.array_equal(a, seq(orc, n, h))


def test_rp_debug_sweep(pip, orc):
    n = 4000
    h = pip.relaxed.make_swap_sequence(n, pip.Rng(91))
    for v in VARIANTS:
        a = np.arange(n, dtype=np.uint64)
        pip.relaxed.random_permutation(a, h, variant=v, debug=True)
        assert np.array_equal(a, seq(orc, n, h))


def test_rp_arbitrary_values(pip, orc):
    # A need not be the identity: any words are permuted
    n = 50_000
    x = rand_words(2, n)
    h = pip.relaxed.make_swap_sequence(n, pip.Rng(8))
    a = dev(x)
    pip.relaxed.random_permutation(a, dev(h))
    want = x.copy()
    orc.seq_knuth_shuffle(want, h)
    assert np.array_equal(host(a), want)


# ----------------------------------------------------------------- merge

def test_merge_examples(pip):
    a = np.array([1, 3, 5, 2, 4, 6], dtype=np.uint64)
    pip.strong.merge_strong(a, 3)
    assert a.tolist() == [1, 2, 3, 4, 5, 6]
    b = np.array([1, 3, 5, 2, 4, 6], dtype=np.uint64)
    pip.relaxed.merge_relaxed(b, 3, pip.EpsilonConfig(0.5, 1e-12))
    assert b.tolist() == [1, 2, 3, 4, 5, 6]


def test_merge_debug_rejects_unsorted(pip):
    with pytest.raises(ValueError, match="unsorted input run"):
        pip.strong.merge_strong(np.array([3, 1, 2, 4], dtype=np.uint64), 2, debug=True)
    with pytest.raises(ValueError, match="unsorted input run"):
        pip.relaxed.merge_relaxed(np.array([2, 1, 3, 4], dtype=np.uint64), 2, debug=True)
    with pytest.raises(ValueError):
        pip.strong.merge_strong(np.arange(4, dtype=np.uint64), 5)


def test_merge_empty_runs(pip):
    x = np.sort(rand_words(8, 100))
    a = x.copy()
    pip.strong.merge_strong(a, 0)
    pip.strong.merge_strong(a, len(a))
    assert np.array_equal(a, x)


def test_merge_golden(pip):
    g = golden("merge")
    for key in g.files:
        if not key.startswith("in_"):
            continue
        name = key[3:]
        x, split, want = g[key], int(g["split_" + name][0]), g["out_" + name]
        a = x.copy()
        pip.strong.merge_strong(a, split)
        assert np.array_equal(a, want), name
        t = dev(x)
        pip.relaxed.merge_relaxed(t, split)
        assert np.array_equal(host(t), want), name


SIZES = [(1, 1), (5, 3), (100, 1), (1, 100), (1000, 1000), (4096, 999), (8192, 8192),
         (8191, 8193), (8193, 1), (1, 8193), (20_000, 13_001), (65_536, 65_536), (100_003, 7),
         (7, 100_003), (300_000, 290_000), (1 << 20, 1 << 20), (1_234_567, 2_345_678)]


@pytest.mark.parametrize("na,nb", SIZES)
@pytest.mark.parametrize("hi", [50, 1 << 30, None])
def test_merge_sizes_vs_oracle(pip, orc, na, nb, hi):
    rng_seed = na * 7919 + nb
    x = np.sort(rand_words(rng_seed, na, hi))
    y = np.sort(rand_words(rng_seed + 1, nb, hi))
    want = orc.seq_merge(x, y)
    a = np.concatenate([x, y])
    t = dev(a)
    pip.strong.merge_strong(t, na)
    assert np.array_equal(host(t), want)
    t = dev(a)
    pip.relaxed.merge_relaxed(t, na)
    assert np.array_equal(host(t), want)


@pytest.mark.parametrize("case", ["a_all_greater", "b_all_greater", "identical", "interleave",
                                  "one_value"])
def test_merge_structured(pip, case):
    n = 8192 * 9 + 123
    na = n // 2
    if case == "a_all_greater":
        x, y = np.arange(na, dtype=np.uint64) + np.uint64(10**9), np.arange(n - na, dtype=np.uint64)
    elif case == "b_all_greater":
        x, y = np.arange(na, dtype=np.uint64), np.arange(n - na, dtype=np.uint64) + np.uint64(10**9)
    elif case == "identical":
        x = np.arange(na, dtype=np.uint64)
        y = np.arange(n - na, dtype=np.uint64)
    elif case == "interleave":
        x = np.arange(na, dtype=np.uint64) * np.uint64(2)
        y = np.arange(n - na, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    else:
        x = np.full(na, 7, dtype=np.uint64)
        y = np.full(n - na, 7, dtype=np.uint64)
    a = np.concatenate([x, y])
    want = np.sort(a)
    for budget in (pip.EpsilonConfig(0.5), pip.EpsilonConfig(0.7, 1e-12)):
        t = dev(a)
        pip.relaxed.merge_relaxed(t, na, budget)
        assert np.array_equal(host(t), want), (case, budget)
    t = dev(a)
    pip.strong.merge_strong(t, na)
    assert np.array_equal(host(t), want)


@pytest.mark.parametrize("eps", [0.3, 0.5, 0.7])
def test_merge_relaxed_within_budget(pip, eps):
    n = 65_536
    cfg = pip.EpsilonConfig(eps, 1e-12)
    b = cfg.prefix_words(n)
    x = rand_words(41, n)
    x[: n // 2].sort()
    x[n // 2:].sort()
    meter = pip.SpaceMeter()
    a = x.copy()
    rep = pip.meter_scope(meter, 8 * b, lambda: pip.relaxed.merge_relaxed(a, n // 2, cfg))
    assert meter.current_words == 0
    assert rep.peak_words <= 8 * b, (eps, rep.peak_words, 8 * b)
    assert np.array_equal(a, np.sort(x))


def test_merge_full_range_unsigned(pip):
    # acceptance 12: full-range words compare unsigned
    rng = np.random.default_rng(12)
    x = np.sort(rng.integers(0, 1 << 64, size=50_000, dtype=np.uint64))
    y = np.sort(rng.integers(0, 1 << 64, size=70_000, dtype=np.uint64))
    a = np.concatenate([x, y])
    t = dev(a)
    pip.relaxed.merge_relaxed(t, len(x))
    assert np.array_equal(host(t), np.sort(a))


@pytest.mark.parametrize("mode", ["0", "1", "2", "3", "3f", "c16", "c8"])
@pytest.mark.parametrize("n,seed,frac,debug", [(100_000, 55, 0.02, False), (1_000_000, 1, 0.02, False),
                                               (20_000, 3, 1e-12, True), (3000, 0, 0.05, True),
                                               (3_000_017, 7, 0.05, False)])
def test_rp_reservation_modes(pip, orc, monkeypatch, mode, n, seed, frac, debug):
    # PIP_RP_BM forces the device reservation scheme: 0 hash table + dense
    # window, 1 bitmaps B/C, 2 bitmap B + collided lists, 3 folded collision
    # bitmap + own band of B + H block counts ("3f": a 1024-bit fold, so most
    # iterates share folded bits with others and go through the list).  All
    # must reproduce the reference's rounds exactly (relaxed.py:176-227).
    # "c16" / "c8": the one-cluster kernel (rp_cluster.cu, 16 or 8 CTAs;
    # it takes only the sizes that fit a cluster's shared memory)
    if mode.startswith("c"):
        monkeypatch.setenv("PIP_RP_CLUSTER", "1" if mode == "c16" else "8")
    else:
        monkeypatch.setenv("PIP_RP_BM", mode[0])
    if mode == "3f":
        monkeypatch.setenv("PIP_RP_FOLD_LOG2", "10")
    h = (np.zeros(n, dtype=np.uint64) if seed == 0
         else pip.relaxed.make_swap_sequence(n, pip.Rng(seed)))
    budget = pip.EpsilonConfig(0.5, frac)
    a = dev(np.arange(n, dtype=np.uint64))
    st = pip.relaxed.random_permutation(a, dev(h), "final", budget, debug=debug)
    b = np.arange(n, dtype=np.uint64)
    ref = orc.ref_random_permutation(b, h, budget.prefix_words(n), "final", threads=8)
    assert np.array_equal(host(a), b)
    assert st.rounds == ref["rounds"]
    assert st.committed_per_round == ref["committed_per_round"]
    assert st.peak_table_load == ref["peak_count"] / ref["capacity"]


@pytest.mark.parametrize("na,nb", [(8192 * 5, 8192 * 4 + 17), (20_000, 13_001), (300_000, 290_000),
                                   (65_536, 65_536), (8193, 30_001)])
@pytest.mark.parametrize("mode", ["offset_view", "mapped_staging", "global_rule", "pointer_jumping"])
def test_merge_staging_layouts(pip, orc, monkeypatch, na, nb, mode):
    """Both staging layouts of the block phase: contiguous sides (interior
    piece boundaries 16-byte aligned) and the segment map (odd word offset of
    the chunk grid, or forced with PIP_MERGE_DBG bit 3); and the global form
    of the dataflow rule (PIP_MERGE_DBG bit 4) beside the per-slot one; and
    pointer jumping for cut-free cycles (bit 5) beside the serial rotation."""
    x = np.sort(rand_words(na + 3 * nb, na, 1 << 20))
    y = np.sort(rand_words(na + 5 * nb, nb, 1 << 20))
    want = orc.seq_merge(x, y)
    a = np.concatenate([x, y])
    if mode == "offset_view":
        buf = dev(np.concatenate([np.zeros(1, dtype=np.uint64), a]))
        t = buf[1:]
    else:
        monkeypatch.setenv("PIP_MERGE_DBG", {"mapped_staging": "8", "global_rule": "16",
                                             "pointer_jumping": "32"}[mode])
        t = dev(a)
    pip.relaxed.merge_relaxed(t, na)
    assert np.array_equal(host(t), want)
    if mode == "offset_view":
        assert int(buf[0].item()) == 0
