"""GPU parity of the streamed host-buffer partition (pip_partition_u64_host):
numpy arrays through strong.partition_unstable, checked against the
reference's contract (strong.py:352-392: m = number of kept words, kept words
in a[:m], the rest in a[m:], same multiset).  Chunks are uploaded from both
ends; chunk boundaries are exercised at the default chunk (2^24 words) and,
in subprocesses, at 2^16 words with 4 and 2 chunks in flight."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def check(pred, before, after, m):
    keep = pred(before)
    assert m == int(np.count_nonzero(keep))
    assert bool(np.all(pred(after[:m]))) and not bool(np.any(pred(after[m:])))
    assert np.array_equal(np.sort(after), np.sort(before))


def inputs(case: str, n: int, seed: int):
    g = np.random.default_rng(seed)
    i = np.arange(n, dtype=np.uint64)
    if case == "random":
        return g.integers(0, 1 << 64, n, dtype=np.uint64)
    if case == "all_true":
        return i * np.uint64(3)
    if case == "all_false":
        return i * np.uint64(3) + np.uint64(1)
    if case == "true_first":
        return np.where(i < n // 3, i * 3, i * 3 + 1).astype(np.uint64)
    if case == "false_first":
        return np.where(i < n // 3, i * 3 + 1, i * 3).astype(np.uint64)
    if case == "sparse":  # ~1% kept
        x = g.integers(0, 1 << 62, n, dtype=np.uint64) * np.uint64(3) + np.uint64(1)
        x[g.random(n) < 0.01] = np.uint64(6)
        return x
    x = g.integers(0, 1 << 62, n, dtype=np.uint64) * np.uint64(3)  # "dense": ~99% kept
    x[g.random(n) < 0.01] = np.uint64(1)
    return x


CASES = ["random", "all_true", "all_false", "true_first", "false_first", "sparse", "dense"]


@pytest.mark.parametrize("case", CASES)
def test_partition_host_default_chunk(case):
    import paper_2103_01216_b200 as pip

    n = 3 * (1 << 24) + 12_345
    x = inputs(case, n, 3)
    a = x.copy()
    p = pip.pred.mod_eq(3, 0)
    m = pip.strong.partition_unstable(a, p)
    check(p, x, a, m)


_SUB = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + "/tests")
import paper_2103_01216_b200 as pip
from test_gpu_partition_host import inputs, check, CASES
p = pip.pred.mod_eq(3, 0)
for case in CASES:
    for n in (65_537, 200_000, 1_000_003, 1 << 20):
        for seed in (1, 2):
            x = inputs(case, n, seed)
            a = x.copy()
            m = pip.strong.partition_unstable(a, p)
            check(p, x, a, m)
q = pip.pred.even()
x = inputs("random", 777_777, 9)
a = x.copy()
check(q, x, a, pip.strong.partition_unstable(a, q))
print("ok")
"""


@pytest.mark.parametrize("env", [{"PIP_HOST_CHUNK_LOG2": "16"},
                                 {"PIP_HOST_CHUNK_LOG2": "16", "PIP_HOST_NBUF": "2"},
                                 {"PIP_HOST_CHUNK_LOG2": "16", "PIP_PARTITION_HOST_INPLACE": "1"}])
def test_partition_host_small_chunks(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", _SUB, str(ROOT)], env=e, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
