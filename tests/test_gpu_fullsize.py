"""Bit-exact parity of BASELINE.json's configs at their FULL sizes.

The kernels run at the benchmark sizes (C1 scan 2^32, C2 filter 2^32,
C3 merge 2 x 2^31, C4 permutation 2^30 — the regime above 2^31 words where
32-bit index bugs live) and every output word is compared with the C
oracle (oracle/pip_oracle.c, restating baselines.py:26-54, 99-114), streamed
in windows so host RAM stays bounded.  Inputs are the bench's own
generators (runtime.Rng on the device, bench.py), regenerated window by
window for the check.  The *_host entry points (the e2e headline path) are
checked the same way at 2^32.

Reference: baselines.seq_scan / seq_filter / seq_merge / seq_knuth_shuffle
(baselines.py:26-54, 99-114); cli.py:263 (the --verify rows).
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.fullsize]

WIN = 1 << 26  # words per compared window (512 MiB)
M64 = (1 << 64) - 1


@pytest.fixture(scope="module")
def pip():
    import torch

    import paper_2103_01216_b200 as pip

    yield pip
    torch.cuda.empty_cache()


@pytest.fixture(autouse=True)
def _free_device():
    import torch

    yield
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def need_host(gib: float):
    import psutil

    avail = psutil.virtual_memory().available / 2**30
    if avail < gib:
        pytest.skip(f"needs {gib:.0f} GiB of host RAM, {avail:.0f} available")


def need_device(gib: float):
    import torch

    free, _ = torch.cuda.mem_get_info()
    if free / 2**30 < gib:
        pytest.skip(f"needs {gib:.0f} GiB of device memory, {free / 2**30:.0f} free")


def host_u64(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


class Pinned:
    """Reusable pinned host windows: D2H at PCIe speed, no per-window allocation."""

    def __init__(self, k: int = 2):
        import torch

        self.bufs = [torch.empty(WIN, dtype=torch.int64, pin_memory=True) for _ in range(k)]

    def get(self, t, slot: int = 0) -> np.ndarray:
        b = self.bufs[slot][: t.numel()]
        b.copy_(t)
        return b.numpy().view(np.uint64)


def sort_run(t, pip):
    """Sort a device run longer than torch.sort's INT_MAX limit: pieces of
    2^30 sorted by torch, then merged in place pairwise with merge_relaxed."""
    import torch

    n, piece = t.numel(), 1 << 30
    for s in range(0, n, piece):
        t[s:s + piece] = torch.sort(t[s:s + piece]).values
    width = piece
    while width < n:
        for s in range(0, n, 2 * width):
            e = min(s + 2 * width, n)
            if s + width < e:
                pip.relaxed.merge_relaxed(t[s:e], width)
        width *= 2


def test_c1_scan_2_32(pip, orc):
    """configs[1]: inclusive scan of 2^32 words Rng(1) >> 44, every word."""
    import torch

    need_device(40)
    n = 1 << 32
    rng = pip.Rng(1)
    a = torch.empty(n, dtype=torch.int64, device="cuda")
    rng.words_device(0, n, shift=44, out=a)
    r = pip.strong.scan_inclusive(a)
    buf = torch.empty(WIN, dtype=torch.int64, device="cuda")
    pin = Pinned()
    carry = 0
    for lo in range(0, n, WIN):
        hi = min(n, lo + WIN)
        x = pin.get(rng.words_device(lo, hi, shift=44, out=buf[: hi - lo]), 0)
        want, _ = orc.seq_scan(x, init=carry, inclusive=True)
        got = pin.get(a[lo:hi], 1)
        assert np.array_equal(got, want), f"window [{lo}, {hi})"
        carry = int(want[-1])
    assert r.total == carry


def test_c2_filter_2_32(pip, orc):
    """configs[2]: stable filter x % 3 == 0 of 2^32 words Rng(1) >> 1: the
    kept count and every word of the packed prefix, in order."""
    import torch

    need_device(40)
    n = 1 << 32
    rng = pip.Rng(1)
    p = pip.pred.mod_eq(3, 0)
    a = torch.empty(n, dtype=torch.int64, device="cuda")
    rng.words_device(0, n, shift=1, out=a)
    m = pip.strong.filter_kway(a, p)
    buf = torch.empty(WIN, dtype=torch.int64, device="cuda")
    pin = Pinned()
    pos = 0
    for lo in range(0, n, WIN):
        hi = min(n, lo + WIN)
        x = pin.get(rng.words_device(lo, hi, shift=1, out=buf[: hi - lo]), 0)
        kept = orc.seq_filter(x, p)
        got = pin.get(a[pos: pos + len(kept)], 1)
        assert np.array_equal(got, kept), f"input window [{lo}, {hi}), output at {pos}"
        pos += len(kept)
    assert m == pos
    assert 0.33 < m / n < 0.34


def _coranks(A, B, ranks):
    """Merge-path co-ranks (ties from A, strong.py:474-488) of many output
    ranks at once: i = #A words among the first r outputs."""
    import torch

    na, nb = A.numel(), B.numel()
    r = torch.tensor(ranks, dtype=torch.int64, device=A.device)
    lo = torch.clamp(r - nb, min=0)
    hi = torch.clamp(r, max=na)
    while bool((lo < hi).any()):
        mid = (lo + hi) // 2
        act = lo < hi
        mi = torch.where(act, mid, torch.zeros_like(mid))
        bj = torch.where(act, r - mi - 1, torch.zeros_like(mid))
        # unsigned compare of int64 words: flip the sign bit
        av = A[mi.clamp(max=na - 1)] ^ (-(1 << 63))
        bv = B[bj.clamp(min=0, max=nb - 1)] ^ (-(1 << 63))
        go = act & (bv >= av)
        lo = torch.where(go, mid + 1, lo)
        hi = torch.where(act & ~go, mid, hi)
    return lo.tolist()


def test_c3_merge_2x2_31(pip, orc):
    """configs[3]: in-place merge of two sorted 2^31-word runs of Rng(1) >> 34
    (heavy duplicates): every output word against the sequential merge of
    the untouched runs."""
    import torch

    need_device(75)
    n, split = 1 << 32, 1 << 31
    a = torch.empty(n, dtype=torch.int64, device="cuda")
    pip.Rng(1).words_device(0, n, shift=34, out=a)
    sort_run(a[:split], pip)
    sort_run(a[split:], pip)
    orig = a.clone()
    pip.relaxed.merge_relaxed(a, split)
    A, B = orig[:split], orig[split:]
    bounds = list(range(0, n, WIN)) + [n]
    ci = _coranks(A, B, bounds)
    pin = Pinned(3)
    for k in range(len(bounds) - 1):
        r0, r1 = bounds[k], bounds[k + 1]
        i0, i1 = ci[k], ci[k + 1]
        j0, j1 = r0 - i0, r1 - i1
        want = orc.seq_merge(pin.get(A[i0:i1], 0), pin.get(B[j0:j1], 1))
        got = pin.get(a[r0:r1], 2)
        assert np.array_equal(got, want), f"output window [{r0}, {r1})"


def test_c3_merge_strong_2x2_31(pip):
    """merge_strong (zero-heap schedule) at C3 size: word for word the same
    output as the relaxed merge on the same runs (which the test above pins
    to the oracle), compared on the device."""
    import torch

    need_device(75)
    n, split = 1 << 32, 1 << 31
    a = torch.empty(n, dtype=torch.int64, device="cuda")
    pip.Rng(3).words_device(0, n, shift=34, out=a)
    sort_run(a[:split], pip)
    sort_run(a[split:], pip)
    b = a.clone()
    pip.strong.merge_strong(a, split)
    pip.relaxed.merge_relaxed(b, split)
    assert torch.equal(a, b)
    assert bool((a[1:] >= a[:-1]).all())  # values < 2^30: signed order = unsigned


def test_c4_random_permutation_2_30(pip, orc):
    """configs[4]: n = 2^30 identity, H = make_swap_sequence(n, Rng(1)) on the
    device; the result equals the sequential Knuth shuffle word for word."""
    import torch

    need_device(40)
    need_host(24)
    n = 1 << 30
    h = torch.empty(n, dtype=torch.int64, device="cuda")
    pip.Rng(1).swaps_device(0, n, out=h)
    a = torch.arange(n, dtype=torch.int64, device="cuda")
    st = pip.relaxed.random_permutation(a, h)
    hh = host_u64(h)
    nonself = int(np.count_nonzero(hh != np.arange(n, dtype=np.uint64)))
    assert st.total_committed == nonself
    want = np.arange(n, dtype=np.uint64)
    orc.seq_knuth_shuffle(want, hh)
    del hh
    got = host_u64(a)
    assert np.array_equal(got, want)


def test_c0_random_permutation_host_pcg64(pip, orc):
    """configs[0] through the host entry point (numpy arrays): n = 10^6, H
    from numpy PCG64(1), uniform in [0, i]; round statistics = the oracle's
    port of the reference's DR rounds."""
    n = 10**6
    g = np.random.Generator(np.random.PCG64(1))
    h = g.integers(0, np.arange(1, n + 1, dtype=np.int64), dtype=np.int64).astype(np.uint64)
    a = np.arange(n, dtype=np.uint64)
    st = pip.relaxed.random_permutation(a, h)
    want = np.arange(n, dtype=np.uint64)
    orc.seq_knuth_shuffle(want, h)
    assert np.array_equal(a, want)
    ref = np.arange(n, dtype=np.uint64)
    info = orc.ref_random_permutation(ref, h, pip.EpsilonConfig(0.5).prefix_words(n))
    assert st.rounds == info["rounds"]
    assert st.committed_per_round == info["committed_per_round"]


def test_scan_host_2_32(pip, orc):
    """pip_scan_u64_host (the e2e path) on a 32 GiB host array: 256 chunks,
    carry handed from chunk to chunk; every word checked."""
    need_host(72)
    import torch

    n = 1 << 32
    x = np.empty(n, dtype=np.uint64)
    rng = pip.Rng(1)
    buf = torch.empty(WIN, dtype=torch.int64, device="cuda")
    pin = Pinned(1)
    for lo in range(0, n, WIN):
        x[lo: lo + WIN] = pin.get(rng.words_device(lo, min(n, lo + WIN), shift=44, out=buf))
    r = pip.strong.scan_inclusive(x)
    carry = 0
    for lo in range(0, n, WIN):
        hi = min(n, lo + WIN)
        src = pin.get(rng.words_device(lo, hi, shift=44, out=buf[: hi - lo]))
        want, _ = orc.seq_scan(src, init=carry, inclusive=True)
        assert np.array_equal(x[lo:hi], want), f"window [{lo}, {hi})"
        carry = int(want[-1])
    assert r.total == carry


def test_filter_host_2_32(pip, orc):
    """pip_filter_u64_host (the e2e path) on a 32 GiB host array: each
    chunk's kept words written back behind the upload front; every kept word
    checked in order."""
    need_host(72)
    import torch

    n = 1 << 32
    x = np.empty(n, dtype=np.uint64)
    rng = pip.Rng(1)
    buf = torch.empty(WIN, dtype=torch.int64, device="cuda")
    pin = Pinned(1)
    for lo in range(0, n, WIN):
        x[lo: lo + WIN] = pin.get(rng.words_device(lo, min(n, lo + WIN), shift=1, out=buf))
    p = pip.pred.mod_eq(3, 0)
    m = pip.strong.filter_kway(x, p)
    pos = 0
    for lo in range(0, n, WIN):
        hi = min(n, lo + WIN)
        kept = orc.seq_filter(pin.get(rng.words_device(lo, hi, shift=1, out=buf[: hi - lo])), p)
        assert np.array_equal(x[pos: pos + len(kept)], kept), f"input window [{lo}, {hi})"
        pos += len(kept)
    assert m == pos
