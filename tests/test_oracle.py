"""Pin the C oracle (oracle/pip_oracle.c) before trusting it:
  * against the golden fixtures produced by the reference itself
    (tests/golden/make_golden.py) — runs everywhere;
  * against the live reference `pipal` on fresh seeded inputs, including the
    reference's own known-answer and exhaustive cases — build container only.
"""
from __future__ import annotations

import itertools

import numpy as np
import pytest

from conftest import golden, rand_words

from paper_2103_01216_b200 import pred as P

VARIANTS = ("naive", "flat", "oneres", "final")


def test_oracle_scan_golden(orc):
    g = golden("scan")
    for key in g.files:
        if key.startswith("in_"):
            name = key[3:]
            out, tot = orc.seq_scan(g[key])
            assert np.array_equal(out, g["out_" + name]) and tot == int(g["tot_" + name][0])
            a = g[key].copy()
            assert orc.ref_scan(a, 4) == tot and np.array_equal(a, g["out_" + name])


def test_oracle_filter_golden(orc):
    g = golden("filter")
    preds = {"even": P.even(), "odd": P.odd(), "mod3": P.mod_eq(3, 0)}
    for key in g.files:
        if key.startswith("out_"):
            pname, name = key[4:].split("_", 1)
            x = g["in_" + name]
            assert np.array_equal(orc.seq_filter(x, preds[pname]), g[key])
            a = x.copy()
            m = orc.ref_filter_kway(a, preds[pname], 4)
            assert m == len(g[key]) and np.array_equal(a[:m], g[key])


def test_oracle_partition_golden(orc):
    # the C port reproduces the reference's partition_unstable word for word
    g = golden("partition")
    preds = {"even": P.even(), "mod3": P.mod_eq(3, 0), "le2e62": P.le(1 << 62)}
    for key in g.files:
        if key.startswith("out_"):
            pname, name = key[4:].split("_", 1)
            a = g["in_" + name].copy()
            m = orc.ref_partition_unstable(a, preds[pname])
            assert m == int(g[f"m_{pname}_{name}"][0]) and np.array_equal(a, g[key])


def test_oracle_merge_golden(orc):
    g = golden("merge")
    for key in g.files:
        if key.startswith("in_"):
            name = key[3:]
            x, split, want = g[key], int(g["split_" + name][0]), g["out_" + name]
            assert np.array_equal(orc.seq_merge(x[:split], x[split:]), want)
            a = x.copy()
            orc.ref_merge_strong(a, split, 4)
            assert np.array_equal(a, want)


def test_oracle_rp_golden(orc):
    """The DR-round port reproduces the reference's rounds, committed counts,
    peak table load and trace for all four variants."""
    g = golden("rp")
    names = sorted({k.split("__")[0] for k in g.files})
    for name in names:
        h = g[name + "__h"]
        n = len(h)
        eps, frac = (float(v) for v in g[name + "__budget"])
        from paper_2103_01216_b200.runtime import EpsilonConfig

        prefix = EpsilonConfig(eps, frac).prefix_words(n)
        a = np.arange(n, dtype=np.uint64)
        r = orc.ref_random_permutation(a, h, prefix, str(g[name + "__variant"][0]), threads=4,
                                       want_trace=True)
        assert np.array_equal(a, g[name + "__out"]), name
        assert r["rounds"] == int(g[name + "__rounds"][0]), name
        assert r["committed_per_round"] == g[name + "__committed"].tolist(), name
        assert r["peak_count"] / r["capacity"] == float(g[name + "__peak"][0]), name
        tr = np.concatenate(r["trace"]) if r["trace"] else np.empty(0, np.uint64)
        assert np.array_equal(tr, g[name + "__trace"]), name
        b = np.arange(n, dtype=np.uint64)
        orc.seq_knuth_shuffle(b, h)
        assert np.array_equal(a, b)


def test_oracle_rng_golden():
    from paper_2103_01216_b200.relaxed import make_swap_sequence
    from paper_2103_01216_b200.runtime import Rng

    g = golden("rng")
    for seed in (0, 1, 177, (1 << 64) - 1):
        assert np.array_equal(Rng(seed).words(5, 5000), g[f"words_{seed}"])
        assert np.array_equal(make_swap_sequence(3000, Rng(seed)), g[f"swaps_{seed}"])


# --------------------------------------------------- live reference (container)

@pytest.mark.reference
def test_oracle_vs_reference_scan_filter_merge(ref, orc):
    rng = np.random.default_rng(7)
    for n in [0, 1, 2, 255, 256, 257, 4096, 12345, 100_003]:
        x = rng.integers(0, 1 << 64, size=n, dtype=np.uint64)
        want, tot = ref.baselines.seq_scan(x)
        out, t2 = orc.seq_scan(x)
        assert np.array_equal(out, want) and t2 == tot
        a = x.copy()
        r = ref.strong.scan(a)
        b = x.copy()
        assert orc.ref_scan(b, 4) == r.total and np.array_equal(a, b)
        for p in (P.even(), P.odd(), P.mod_eq(3, 0), P.lt(1 << 62)):
            a = x.copy()
            m = ref.strong.filter_kway(a, p)
            assert np.array_equal(orc.seq_filter(x, p), a[:m])
            assert np.array_equal(ref.baselines.seq_filter(x, p), a[:m])
        na = n // 3
        xs = np.sort(rng.integers(0, 40, size=na, dtype=np.uint64))
        ys = np.sort(rng.integers(0, 40, size=n - na, dtype=np.uint64))
        assert np.array_equal(orc.seq_merge(xs, ys), ref.baselines.seq_two_finger_merge(xs, ys))
    # generic ops (test_strong.py:104-107)
    a = np.array([2, 9, 1, 5], dtype=np.uint64)
    out, tot = orc.seq_scan(a, op="max")
    r = ref.strong.scan(a, op=max, identity=0)
    assert out.tolist() == a.tolist() and tot == r.total


@pytest.mark.reference
@pytest.mark.parametrize("variant", VARIANTS)
def test_oracle_rp_exhaustive_vs_reference(ref, orc, variant):
    # every valid H for n <= 6 (test_acceptance.py:128-145), full prefix
    cfg = ref.runtime.EpsilonConfig(0.5, prefix_fraction=1.0)
    for n in range(1, 7):
        for tail in itertools.product(*(range(i + 1) for i in range(1, n))):
            h = np.array((0,) + tail, dtype=np.uint64)
            a = np.arange(n, dtype=np.uint64)
            st = ref.relaxed.random_permutation(a, h, variant, cfg)
            b = np.arange(n, dtype=np.uint64)
            r = orc.ref_random_permutation(b, h, cfg.prefix_words(n), variant)
            assert np.array_equal(a, b) and st.rounds == r["rounds"]
            assert st.committed_per_round == r["committed_per_round"]


@pytest.mark.reference
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("n,seed,eps,frac", [(10_000, 177, 0.5, 0.02), (100_000, 55, 0.5, 0.02),
                                             (30_000, 5, 0.3, 1e-12), (7_777, 8, 0.7, 1e-12)])
def test_oracle_rp_rounds_vs_reference(ref, orc, variant, n, seed, eps, frac):
    h = ref.relaxed.make_swap_sequence(n, ref.runtime.Rng(seed))
    cfg = ref.runtime.EpsilonConfig(eps, frac)
    a = np.arange(n, dtype=np.uint64)
    tr = []
    st = ref.relaxed.random_permutation(a, h, variant, cfg, trace=tr)
    b = np.arange(n, dtype=np.uint64)
    r = orc.ref_random_permutation(b, h, cfg.prefix_words(n), variant, threads=8, want_trace=True)
    assert np.array_equal(a, b)
    assert st.rounds == r["rounds"] and st.committed_per_round == r["committed_per_round"]
    assert st.peak_table_load == r["peak_count"] / r["capacity"]
    assert all(np.array_equal(x, y) for x, y in zip(tr, r["trace"]))


@pytest.mark.reference
def test_oracle_knuth_vs_reference(ref, orc):
    for n, seed in [(1, 1), (2, 2), (1000, 3), (65_536, 4)]:
        h = ref.relaxed.make_swap_sequence(n, ref.runtime.Rng(seed))
        a = np.arange(n, dtype=np.uint64)
        ref.baselines.seq_knuth_shuffle(a, h)
        b = np.arange(n, dtype=np.uint64)
        orc.seq_knuth_shuffle(b, h)
        assert np.array_equal(a, b)
    # the reference's double-entry check (test_baselines.py:32-50): composition
    x = rand_words(5, 300)
    h = ref.relaxed.make_swap_sequence(300, ref.runtime.Rng(11))
    y = x.copy()
    orc.seq_knuth_shuffle(y, h)
    assert sorted(y.tolist()) == sorted(x.tolist())
