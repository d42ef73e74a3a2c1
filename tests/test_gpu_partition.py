"""GPU parity: unstable in-place partition (strong.partition_unstable,
relaxed.partition_relaxed) against the reference's contract and known
answers (test_strong.py:189-207): m == #true, a[0:m) all true, a[m:n) all
false, the multiset preserved.  The reference's order inside each side is
unspecified (its tests check exactly these properties)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, rand_words

pytestmark = pytest.mark.gpu


def dev(a: np.ndarray):
    import torch

    return torch.from_numpy(a.view(np.int64).copy()).cuda()


def host(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


@pytest.fixture(scope="module")
def pip():
    import paper_2103_01216_b200 as pip

    return pip


def check(pred, before: np.ndarray, after: np.ndarray, m: int) -> None:
    keep = np.asarray(pred(before), dtype=bool)
    assert m == int(np.count_nonzero(keep))
    assert np.all(np.asarray(pred(after[:m]), dtype=bool))
    assert not np.any(np.asarray(pred(after[m:]), dtype=bool))
    assert np.array_equal(np.sort(after), np.sort(before))


def test_partition_known_answers(pip):
    # test_strong.py:189-197
    a = np.array([1, 2, 3, 4], dtype=np.uint64)
    m = pip.strong.partition_unstable(a, pip.pred.le(2))
    assert m == 2 and sorted(a[:2].tolist()) == [1, 2] and sorted(a[2:].tolist()) == [3, 4]
    b = np.array([5, 7, 9], dtype=np.uint64)
    assert pip.strong.partition_unstable(b, pip.pred.lt(0)) == 0
    assert sorted(b.tolist()) == [5, 7, 9]
    assert pip.strong.partition_unstable(np.zeros(0, dtype=np.uint64), pip.pred.even()) == 0


SIZES = [1, 2, 17, 1000, 4095, 4096, 4097, 8191, 8193, 30_000, 65_536, 100_003, 1_000_003]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("which", ["even", "mod3", "lt1pct", "lt99pct"])
def test_partition_device_vs_contract(pip, n, which):
    x = rand_words(n * 3 + 7, n)
    p = {"even": pip.pred.even(), "mod3": pip.pred.mod_eq(3, 0),
         "lt1pct": pip.pred.lt(1 << 57), "lt99pct": pip.pred.lt((1 << 64) - (1 << 57))}[which]
    t = dev(x)
    m = pip.strong.partition_unstable(t, p)
    check(p, x, host(t), m)


@pytest.mark.parametrize("n", [0, 1, 17, 1000, 30_000])
def test_partition_host_arrays(pip, n):
    # test_strong.py:200-207 (numpy in, numpy out)
    a = rand_words(n + 3, n)
    ref = a.copy()
    m = pip.strong.partition_unstable(a, pip.pred.even())
    check(pip.pred.even(), ref, a, m)


@pytest.mark.parametrize("case", ["all_true", "all_false", "sorted_true_first",
                                  "sorted_false_first", "alternating"])
def test_partition_structured(pip, case):
    n = 4096 * 7 + 321
    i = np.arange(n, dtype=np.uint64)
    x = {"all_true": i * np.uint64(2), "all_false": i * np.uint64(2) + np.uint64(1),
         "sorted_true_first": np.where(i < n // 3, i * 2, i * 2 + 1).astype(np.uint64),
         "sorted_false_first": np.where(i < n // 3, i * 2 + 1, i * 2).astype(np.uint64),
         "alternating": i}[case]
    p = pip.pred.even()
    t = dev(x)
    m = pip.strong.partition_unstable(t, p)
    out = host(t)
    check(p, x, out, m)
    if case in ("all_true", "all_false", "sorted_true_first"):
        assert np.array_equal(out, x)  # nothing misplaced: nothing moves


def test_partition_prefix_n_and_view(pip):
    x = rand_words(5, 50_000)
    buf = dev(np.concatenate([np.zeros(1, dtype=np.uint64), x]))
    t = buf[1:]  # odd word offset
    m = pip.strong.partition_unstable(t, pip.pred.mod_eq(5, 2), n=40_000)
    out = host(t)
    check(pip.pred.mod_eq(5, 2), x[:40_000], out[:40_000], m)
    assert np.array_equal(out[40_000:], x[40_000:]) and int(buf[0].item()) == 0


@pytest.mark.parametrize("eps", [0.3, 0.5, 0.7])
def test_partition_relaxed_budget_and_rounds(pip, eps):
    # relaxed.py:312-344: same contract, rounds of b(n) words, charged <= 8 b
    n = 65_536
    cfg = pip.EpsilonConfig(eps, 1e-12)
    b = cfg.prefix_words(n)
    x = rand_words(41, n)
    a = x.copy()
    meter = pip.SpaceMeter()
    sink: list = []
    got = []
    rep = pip.meter_scope(meter, 8 * b, lambda: got.append(pip.relaxed.partition_relaxed(
        a, pip.pred.odd(), cfg, stats_sink=sink)))
    assert meter.current_words == 0 and 0 < rep.peak_words <= 8 * b
    check(pip.pred.odd(), x, a, got[0])
    assert sink[0].rounds == -(-n // b) and sum(sink[0].committed_per_round) == n


def test_partition_golden(pip):
    # the reference's own outputs (tests/golden/make_golden.py): same m, same
    # multiset on each side
    g = golden("partition")
    preds = {"even": pip.pred.even(), "mod3": pip.pred.mod_eq(3, 0), "le2e62": pip.pred.le(1 << 62)}
    for key in g.files:
        if key.startswith("out_"):
            pname, name = key[4:].split("_", 1)
            x = g["in_" + name]
            m_ref = int(g[f"m_{pname}_{name}"][0])
            t = dev(x)
            m = pip.strong.partition_unstable(t, preds[pname])
            out = host(t)
            assert m == m_ref
            assert np.array_equal(np.sort(out[:m]), np.sort(g[key][:m]))
            assert np.array_equal(np.sort(out[m:]), np.sort(g[key][m:]))


# ----------------------------------------------------------------- quicksort

@pytest.mark.parametrize("n", [0, 1, 3, 100, 10_000, 50_000])
def test_quicksort_strong_matches_sorted(pip, n):
    # test_strong.py:210-215 (host arrays)
    a = rand_words(n + 1, n)
    ref = np.sort(a)
    pip.strong.quicksort_strong(a, pip.Rng(31))
    assert np.array_equal(a, ref)


def test_quicksort_duplicates(pip):
    # test_strong.py:218-221
    a = np.array([3, 1, 2] * 500, dtype=np.uint64)
    pip.strong.quicksort_strong(a, pip.Rng(5))
    assert np.array_equal(a, np.sort(np.array([3, 1, 2] * 500, dtype=np.uint64)))


@pytest.mark.parametrize("case", ["random", "few_values", "all_equal", "sorted", "reversed",
                                  "full_range_max"])
def test_quicksort_device_large(pip, case):
    n = 1_000_003
    rng = np.random.default_rng(7)
    x = {"random": rng.integers(0, 1 << 64, size=n, dtype=np.uint64),
         "few_values": rng.integers(0, 5, size=n, dtype=np.uint64),
         "all_equal": np.full(n, 42, dtype=np.uint64),
         "sorted": np.arange(n, dtype=np.uint64),
         "reversed": np.arange(n, dtype=np.uint64)[::-1].copy(),
         "full_range_max": np.where(rng.random(n) < 0.1, np.uint64((1 << 64) - 1),
                                    rng.integers(0, 1 << 64, size=n, dtype=np.uint64))}[case]
    t = dev(x)
    pip.strong.quicksort_strong(t, pip.Rng(9))
    assert np.array_equal(host(t), np.sort(x))


def test_quicksort_relaxed_metered(pip):
    n = 300_000
    x = rand_words(77, n)
    a = x.copy()
    meter = pip.SpaceMeter()
    cfg = pip.EpsilonConfig(0.5)
    b = cfg.prefix_words(n)
    rep = pip.meter_scope(meter, 8 * b, lambda: pip.relaxed.quicksort_relaxed(a, pip.Rng(3), cfg))
    assert meter.current_words == 0 and rep.peak_words <= 8 * b
    assert np.array_equal(a, np.sort(x))


def test_sort_segments_ragged(pip):
    # the quicksort base case (strong.py:453-454) on its own: disjoint ragged
    # segments of 2 .. 2^20 words (one and several shared-memory chunks,
    # non-powers of two), words between them untouched
    import ctypes as C

    import torch

    from paper_2103_01216_b200 import _lib

    lens = [2, 3, 255, 8191, 8192, 8193, 12345, 16384, 40000, 65535, 65536, 1, 262147, 1 << 20]
    gap = 7
    los, pos = [], 0
    for ln in lens:
        los.append(pos)
        pos += ln + gap
    rng = np.random.default_rng(11)
    x = rng.integers(0, 1 << 64, size=pos, dtype=np.uint64)
    x[: pos // 3] = rng.integers(0, 4, size=pos // 3, dtype=np.uint64)
    x[pos // 2: pos // 2 + 5000] = np.uint64((1 << 64) - 1)
    ref = x.copy()
    for lo, ln in zip(los, lens):
        ref[lo: lo + ln] = np.sort(ref[lo: lo + ln])
    t = dev(x)
    slo = torch.tensor(los, dtype=torch.int64, device="cuda")
    sln = torch.tensor(lens, dtype=torch.int32, device="cuda")
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    assert lib.pip_sort_segments_u64(t.data_ptr(), slo.data_ptr(), sln.data_ptr(),
                                     C.c_uint64(len(lens)), st) == 0
    assert np.array_equal(host(t), ref)


@pytest.mark.parametrize("big", [1 << 13, (1 << 16) + 3, (1 << 21) + 5])
def test_sort_segments_grid_ragged(pip, big):
    # the grid-wide leaf sort (pip_sort_segments_grid_u64): ragged segments
    # below, at and above one chunk next to one long segment
    import ctypes as C

    import torch

    from paper_2103_01216_b200 import _lib

    lens = [2, 3, 255, 8191, 8192, 8193, 40000, 1, big, 65536, 5]
    los, pos = [], 0
    for ln in lens:
        los.append(pos)
        pos += ln + 3
    rng = np.random.default_rng(big)
    x = rng.integers(0, 1 << 64, size=pos, dtype=np.uint64)
    x[: pos // 4] = rng.integers(0, 3, size=pos // 4, dtype=np.uint64)
    x[pos // 2: pos // 2 + 3000] = np.uint64((1 << 64) - 1)
    ref = x.copy()
    for lo, ln in zip(los, lens):
        ref[lo: lo + ln] = np.sort(ref[lo: lo + ln])
    t = dev(x)
    slo = torch.tensor(los, dtype=torch.int64, device="cuda")
    sln = torch.tensor(lens, dtype=torch.int32, device="cuda")
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    assert lib.pip_sort_segments_grid_u64(t.data_ptr(), slo.data_ptr(), sln.data_ptr(),
                                          C.c_uint64(len(lens)), C.c_uint64(max(lens)), st) == 0
    assert np.array_equal(host(t), ref)


@pytest.mark.parametrize("leaf", [8192, 65536, 1 << 19])
@pytest.mark.parametrize("case", ["random", "few_values", "full_range_max"])
def test_quicksort_recursion_small_leaves(pip, monkeypatch, leaf, case):
    # the level-batched recursion itself (many levels of partitions) at leaf
    # sizes below the default
    monkeypatch.setattr(pip.strong, "QS_LEAF", leaf)
    n = 3_000_017
    rng = np.random.default_rng(leaf + len(case))
    x = {"random": rng.integers(0, 1 << 64, size=n, dtype=np.uint64),
         "few_values": rng.integers(0, 7, size=n, dtype=np.uint64),
         "full_range_max": np.where(rng.random(n) < 0.2, np.uint64((1 << 64) - 1),
                                    rng.integers(0, 1 << 64, size=n, dtype=np.uint64))}[case]
    t = dev(x)
    pip.strong.quicksort_strong(t, pip.Rng(13))
    assert np.array_equal(host(t), np.sort(x))


def test_quicksort_above_default_leaf(pip):
    n = (1 << 23) + 11
    x = pip.Rng(21).words(0, n) >> np.uint64(20)
    t = dev(x)
    pip.strong.quicksort_strong(t, pip.Rng(4))
    assert np.array_equal(host(t), np.sort(x))
