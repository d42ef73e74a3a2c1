"""GPU parity: scan / reduce / rotate / filter against the C oracle and the
reference's golden vectors (bit-exact: integer work)."""
from __future__ import annotations

import operator

import numpy as np
import pytest

from conftest import golden, rand_words

pytestmark = pytest.mark.gpu

M64 = (1 << 64) - 1


def dev(a: np.ndarray):
    import torch

    return torch.from_numpy(a.view(np.int64).copy()).cuda()


def host(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


@pytest.fixture(scope="module")
def pip():
    import paper_2103_01216_b200 as pip

    return pip


# ----------------------------------------------------------------- scan

def test_scan_known_answers(pip):
    S = pip.strong
    a = np.array([7], dtype=np.uint64)
    r = S.scan(a)
    assert a.tolist() == [0] and r.total == 7
    a = np.array([1, 1, 1, 1], dtype=np.uint64)
    r = S.scan(a)
    assert a.tolist() == [0, 1, 2, 3] and r.total == 4
    a = np.array([3, 1, 4, 1, 5, 9, 2, 6], dtype=np.uint64)
    r = S.scan(a)
    assert r.total == 31 and a.tolist() == [0, 3, 4, 8, 9, 14, 23, 25]
    a = np.array([M64, 5], dtype=np.uint64)  # wrap (test_baselines.py:20-23)
    r = S.scan(a)
    assert a.tolist() == [0, M64] and r.total == 4
    a = np.array([2, 9, 1, 5], dtype=np.uint64)  # op=max (test_strong.py:104-107)
    r = S.scan(a, op=max, identity=0)
    assert a.tolist() == [0, 2, 9, 9] and r.total == 9
    e = np.empty(0, dtype=np.uint64)
    assert S.scan(e).total == 0 and S.scan(e, identity=5).total == 5


def test_scan_golden(pip):
    g = golden("scan")
    for key in g.files:
        if not key.startswith("in_"):
            continue
        name = key[3:]
        x = g[key]
        want, tot = g["out_" + name], int(g["tot_" + name][0])
        for mode in ("host", "device"):
            if mode == "host":
                a = x.copy()
                r = pip.strong.scan(a)
                got = a
            else:
                t = dev(x)
                r = pip.strong.scan(t)
                got = host(t)
            assert np.array_equal(got, want), (name, mode)
            assert r.total == tot


@pytest.mark.parametrize("n", [2, 3, 255, 256, 257, 511, 512, 1000, 4096, 8191, 8192, 8193,
                               12345, 65536, 100_001, 1 << 20, 3_000_017])
@pytest.mark.parametrize("inclusive", [False, True])
def test_scan_sizes_vs_oracle(pip, orc, n, inclusive):
    x = rand_words(n, n)
    want, tot = orc.seq_scan(x, inclusive=inclusive)
    t = dev(x)
    fn = pip.strong.scan_inclusive if inclusive else pip.strong.scan
    r = fn(t)
    assert np.array_equal(host(t), want)
    assert r.total == tot


@pytest.mark.parametrize("op,name", [(max, "max"), (min, "min"), (operator.xor, "xor"),
                                     (operator.add, "add")])
@pytest.mark.parametrize("n", [1, 5, 1000, 70_000])
def test_scan_generic_ops(pip, orc, op, name, n):
    x = rand_words(n + 3, n)
    for ident in (0, 12345, M64):
        want, tot = orc.seq_scan(x, op=name, init=ident)
        t = dev(x)
        r = pip.strong.scan(t, op=op, identity=ident)
        assert np.array_equal(host(t), want), (name, ident)
        assert r.total == tot


def test_scan_misaligned_view(pip, orc):
    # a view that starts 8 bytes into an allocation takes the scalar path
    import torch

    x = rand_words(9, 50_001)
    base = torch.zeros(50_002, dtype=torch.int64, device="cuda")
    base[1:] = torch.from_numpy(x.view(np.int64)).cuda()
    view = base[1:]
    r = pip.strong.scan(view)
    want, tot = orc.seq_scan(x)
    assert np.array_equal(host(view), want) and r.total == tot
    assert int(base[0].item()) == 0


def test_scan_blocked_identical(pip):
    for n in [1, 5, 255, 256, 1000, 65536, 100_001]:
        x = rand_words(n, n)
        a1, a2 = dev(x), dev(x)
        r1, r2 = pip.strong.scan(a1), pip.strong.scan_blocked(a2)
        assert np.array_equal(host(a1), host(a2)) and r1.total == r2.total


def test_scan_reconstruction(pip):
    orig = rand_words(9, 5000)
    a = orig.copy()
    res = pip.strong.scan(a)
    rec = np.empty_like(a)
    rec[:-1] = a[1:] - a[:-1]
    rec[-1] = np.uint64((res.total - int(a[-1])) & M64)
    assert np.array_equal(rec, orig)


def test_scan_acceptance_small_random(pip, orc):
    rng = np.random.default_rng(1)
    for _ in range(200):
        n = int(rng.integers(1, 1001))
        x = rng.integers(0, 1 << 64, size=n, dtype=np.uint64)
        t = dev(x)
        r = pip.strong.scan(t)
        want, tot = orc.seq_scan(x)
        assert np.array_equal(host(t), want) and r.total == tot


def test_reduce(pip):
    x = rand_words(1, 100_000)
    assert pip.strong.reduce(dev(x)) == int(np.sum(x, dtype=np.uint64))
    assert pip.strong.reduce(np.arange(1, 101, dtype=np.uint64)) == 5050
    assert pip.strong.reduce(np.empty(0, dtype=np.uint64)) == 0
    assert pip.strong.reduce(np.array([3, 9, 1, 7], dtype=np.uint64), op=max) == 9


def test_type_errors(pip):
    with pytest.raises(TypeError):
        pip.strong.scan(np.arange(5, dtype=np.int64))
    with pytest.raises(TypeError):
        pip.strong.scan(np.arange(10, dtype=np.uint64)[::2])
    with pytest.raises(TypeError):
        pip.strong.scan(np.arange(5, dtype=np.uint64), op=lambda a, b: a)
    with pytest.raises(TypeError):
        pip.strong.filter_kway(np.arange(5, dtype=np.uint64), lambda b: b > 1)


# ----------------------------------------------------------------- rotate

@pytest.mark.parametrize("n", [0, 1, 2, 5, 800, 100_003])
def test_rotate(pip, n):
    x = rand_words(n, n)
    for o in sorted({0, min(1, n), n // 3, n // 2, max(n - 1, 0), n}):
        t = dev(x)
        pip.strong.rotate(t, o)
        assert np.array_equal(host(t), np.roll(x, -o))
    a = np.array([1, 2, 3, 4, 5], dtype=np.uint64)
    pip.strong.rotate(a, 2)
    assert a.tolist() == [3, 4, 5, 1, 2]
    with pytest.raises(ValueError):
        pip.strong.rotate(a, 6)


# ----------------------------------------------------------------- filter

def test_filter_examples(pip):
    P = pip.pred
    a = np.array([5, 2, 7, 4], dtype=np.uint64)
    m = pip.strong.filter_kway(a, P.even())
    assert m == 2 and a[:2].tolist() == [2, 4]
    b = np.array([2, 4, 6], dtype=np.uint64)
    assert pip.strong.filter_kway(b, P.even()) == 3 and b.tolist() == [2, 4, 6]


def test_filter_golden(pip):
    g = golden("filter")
    P = pip.pred
    preds = {"even": P.even(), "odd": P.odd(), "mod3": P.mod_eq(3, 0)}
    for key in g.files:
        if not key.startswith("out_"):
            continue
        pname, name = key[4:].split("_", 1)
        x = g["in_" + name]
        want = g[key]
        for mode in ("host", "device"):
            if mode == "host" or len(x) == 0:
                a = x.copy()
                m = pip.strong.filter_kway(a, preds[pname])
                got = a[:m]
            else:
                t = dev(x)
                m = pip.strong.filter_kway(t, preds[pname])
                got = host(t)[:m]
            assert m == len(want) and np.array_equal(got, want), (key, mode)


@pytest.mark.parametrize("n", [0, 1, 10, 1000, 9999, 65536, 8192 * 37 + 5, 2_000_003])
def test_filter_sizes_vs_oracle(pip, orc, n):
    P = pip.pred
    x = rand_words(n + 17, n)
    for p in (P.even(), P.odd(), P.mod_eq(3, 0), P.mod_eq(7, 3), P.mod_eq(1 << 20, 5),
              P.lt(1 << 63), P.ge(3 << 62), P.eq(int(x[0]) if n else 1), P.always(),
              ~P.mod_eq(3, 0), P.bit_set(40), P.mod_eq(1000000007, 17)):
        want = orc.seq_filter(x, p)
        t = dev(x)
        m = pip.strong.filter_kway(t, p)
        assert m == len(want), p
        assert np.array_equal(host(t)[:m], want), p


def test_filter_mod_magic_divisors(pip):
    # the kernel divides by an invariant with u64 magic numbers: check many divisors
    P = pip.pred
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.integers(0, 1 << 64, size=20000, dtype=np.uint64),
                        np.array([0, 1, 2, M64, M64 - 1, 1 << 63, (1 << 63) - 1], dtype=np.uint64)])
    divisors = [1, 2, 3, 5, 6, 7, 10, 11, 12, 13, 25, 100, 641, 1 << 32, (1 << 32) + 1,
                6700417, 1000000007, (1 << 63) + 1, M64, M64 - 2, 3 << 61]
    for d in divisors:
        for r in (0, 1 % d):
            p = P.mod_eq(d, r)
            want = x[(x % np.uint64(d)) == np.uint64(r)]
            t = dev(x)
            m = pip.strong.filter_kway(t, p)
            assert m == len(want) and np.array_equal(host(t)[:m], want), d


def test_filter_stability_small_random(pip, orc):
    P = pip.pred
    rng = np.random.default_rng(99)
    for _ in range(300):
        n = int(rng.integers(0, 120))
        x = rng.integers(0, 8, size=n, dtype=np.uint64)
        t = dev(x) if n else None
        if n == 0:
            assert pip.strong.filter_kway(x.copy(), P.odd()) == 0
            continue
        m = pip.strong.filter_kway(t, P.odd())
        assert host(t)[:m].tolist() == orc.seq_filter(x, P.odd()).tolist()


def test_filter_n_argument(pip, orc):
    P = pip.pred
    x = rand_words(4, 10_000)
    t = dev(x)
    m = pip.strong.filter_kway(t, P.even(), n=7000)
    want = orc.seq_filter(x[:7000], P.even())
    got = host(t)
    assert m == len(want) and np.array_equal(got[:m], want)
    assert np.array_equal(got[7000:], x[7000:])


def test_filter_relaxed_equals_kway(pip):
    P = pip.pred
    for n in [0, 1, 100, 4096, 65_537]:
        x = rand_words(n + 11, n)
        a1, a2 = x.copy(), x.copy()
        m1 = pip.strong.filter_kway(a1, P.even())
        sink = []
        cfg = pip.EpsilonConfig(0.5, 1e-12)
        m2 = pip.relaxed.filter_relaxed(a2, P.even(), cfg, stats_sink=sink)
        assert m1 == m2 and np.array_equal(a1[:m1], a2[:m2])
        if n:  # the device ran the reference's rounds: ceil(n / b) blocks of b words
            b = cfg.prefix_words(n)
            assert sink[0].committed_per_round == [min(b, n - s) for s in range(0, n, b)]
    # device tensor, BASELINE's predicate, several block sizes
    x = rand_words(5, 300_001)
    for frac in (0.02, 0.3, 1.0):
        t = dev(x)
        m = pip.relaxed.filter_relaxed(t, P.mod_eq(3, 0), pip.EpsilonConfig(0.5, frac))
        want = x[(x % np.uint64(3)) == 0]
        assert m == len(want) and np.array_equal(host(t)[:m], want)


# Tile geometry of the default split-role kernels: 13 compute warps x 512 words
# = 6656-word tiles, 4 stages, one CTA per SM; sizes around whole waves of
# tiles (148 x 6656) and single tiles exercise the tail hand-off to the
# register kernel and the carry between them.
WS2_TILE = 13 * 512


@pytest.mark.parametrize("n", [8 * WS2_TILE - 1, 8 * WS2_TILE, 8 * WS2_TILE + 1,
                               148 * WS2_TILE, 148 * WS2_TILE + 7, 3 * 148 * WS2_TILE - 1])
def test_scan_ws2_tile_boundaries(pip, orc, n):
    x = rand_words(n + 1, n, hi=1 << 40)
    for inclusive in (False, True):
        want, tot = orc.seq_scan(x, inclusive=inclusive)
        t = dev(x)
        r = (pip.strong.scan_inclusive if inclusive else pip.strong.scan)(t)
        assert np.array_equal(host(t), want) and r.total == tot, (n, inclusive)


@pytest.mark.parametrize("n", [8 * WS2_TILE - 1, 8 * WS2_TILE + 1, 148 * WS2_TILE + 7,
                               2 * 148 * WS2_TILE - 3])
def test_filter_ws2_tile_boundaries(pip, orc, n):
    P = pip.pred
    x = rand_words(n + 2, n)
    for p in (P.mod_eq(3, 0), P.mod_eq(5, 2), P.mod_eq(8, 1), P.always(), ~P.always(), P.lt(1 << 62),
              ~P.mod_eq(5, 2), ~P.mod_eq(8, 1), ~P.even(), ~P.lt(1 << 62), ~P.mod_eq(3, 0)):
        want = orc.seq_filter(x, p)
        t = dev(x)
        m = pip.strong.filter_kway(t, p)
        assert m == len(want) and np.array_equal(host(t)[:m], want), (n, p)
