"""The checks bench.py runs on its own outputs (they guard the headline
numbers): the merge-path co-rank helper against brute force, and the
sampled-window merge check accepting a correct merge and rejecting a
corrupted one.  CPU tensors, no GPU needed."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def _brute_corank(a, b, r):
    # smallest i with i + j = r and not (j > 0 and i < na and b[j-1] >= a[i])
    na, nb = len(a), len(b)
    for i in range(max(0, r - nb), min(r, na) + 1):
        j = r - i
        if not (j > 0 and i < na and b[j - 1] >= a[i]):
            return i
    raise AssertionError


@pytest.mark.parametrize("seed,hi", [(1, 5), (2, 1000), (3, 1 << 63)])
def test_merge_coranks_matches_brute_force(seed, hi):
    rng = np.random.default_rng(seed)
    a = np.sort(rng.integers(0, hi, size=137, dtype=np.uint64))
    b = np.sort(rng.integers(0, hi, size=91, dtype=np.uint64))
    A = torch.from_numpy(a.view(np.int64))
    B = torch.from_numpy(b.view(np.int64))
    ranks = list(range(0, len(a) + len(b) + 1))
    got = bench.merge_coranks(A, B, ranks, torch)
    assert got == [_brute_corank(a, b, r) for r in ranks]


def test_merge_window_check_accepts_and_rejects(orc):
    rng = np.random.default_rng(4)
    n, na = 1 << 16, (1 << 15) + 3
    a = np.sort(rng.integers(0, 50, size=na, dtype=np.uint64))
    b = np.sort(rng.integers(0, 50, size=n - na, dtype=np.uint64))
    orig = torch.from_numpy(np.concatenate([a, b]).view(np.int64))
    merged = torch.from_numpy(np.sort(np.concatenate([a, b])).view(np.int64))
    bench.check_merge_windows(merged, orig, na, torch)
    bad = merged.clone()
    bad[n // 2] += 1  # one word off in the middle window
    with pytest.raises(AssertionError, match="merge parity"):
        bench.check_merge_windows(bad, orig, na, torch)


def test_windows_cover_start_middle_end():
    w = bench._windows(10_000_000)
    assert w[0][0] == 0 and w[-1][1] == 10_000_000 and len(w) == 3
    assert bench._windows(100) == [(0, 100)]
