"""GPU parity of the streamed host-buffer merge (pip_merge_u64_host): numpy
arrays through strong.merge_strong / relaxed.merge_relaxed, checked against
np.sort of the same words (the reference's contract, strong.py:462-522:
the output is the sorted multiset).  Chunk boundaries are exercised both
at the default chunk (2^24 words) and, in a subprocess, at 2^16."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def runs(case: str, na: int, nb: int, seed: int):
    g = np.random.default_rng(seed)
    if case == "dups":
        x, y = g.integers(0, 1 << 10, na), g.integers(0, 1 << 10, nb)
    elif case == "a_below":
        x, y = g.integers(0, 1 << 20, na), g.integers(1 << 20, 1 << 21, nb)
    elif case == "a_above":
        x, y = g.integers(1 << 40, 1 << 41, na), g.integers(0, 1 << 20, nb)
    elif case == "equal":
        x, y = np.full(na, 7), np.full(nb, 7)
    elif case == "full":
        x = g.integers(0, 1 << 64, na, dtype=np.uint64)
        y = g.integers(0, 1 << 64, nb, dtype=np.uint64)
    else:  # interleaved blocks: long stretches from each side
        x = (np.arange(na) // 4096) * 2 * 4096 + np.arange(na) % 4096
        y = (np.arange(nb) // 4096) * 2 * 4096 + 4096 + np.arange(nb) % 4096
    a = np.concatenate([np.sort(np.asarray(x, dtype=np.uint64)),
                        np.sort(np.asarray(y, dtype=np.uint64))])
    return a


CASES = ["dups", "a_below", "a_above", "equal", "full", "blocks"]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("na,nb", [((1 << 24) + 12_345, (1 << 24) + 3), (3, (1 << 25) + 1),
                                   ((1 << 25) + 7, 5)])
def test_host_merge_default_chunk(case, na, nb):
    import paper_2103_01216_b200 as pip

    a = runs(case, na, nb, 11)
    want = np.sort(a)
    if case in ("dups", "full"):
        pip.strong.merge_strong(a, na)
    else:
        pip.relaxed.merge_relaxed(a, na)
    assert np.array_equal(a, want)


_SUB = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + "/tests")
import paper_2103_01216_b200 as pip
from test_gpu_merge_host import runs, CASES
for case in CASES:
    for na, nb in [(1, 1), (1, 70_000), (70_000, 1), (65_536, 65_536), (300_001, 411_113),
                   (1_000_003, 17), (17, 1_000_003), (131_071, 131_073)]:
        for seed in (1, 2):
            a = runs(case, na, nb, seed)
            want = np.sort(a)
            pip.relaxed.merge_relaxed(a, na)
            assert np.array_equal(a, want), (case, na, nb, seed)
            b = runs(case, na, nb, seed)
            pip.strong.merge_strong(b, na)
            assert np.array_equal(b, want), (case, na, nb, seed)
print("ok")
"""


@pytest.mark.parametrize("env", [{"PIP_HOST_CHUNK_LOG2": "16"},
                                 {"PIP_HOST_CHUNK_LOG2": "16", "PIP_HOST_NBUF": "2"},
                                 {"PIP_MERGE_HOST_INPLACE": "1"}])
def test_host_merge_small_chunks(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", _SUB, str(ROOT)], env=e, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
