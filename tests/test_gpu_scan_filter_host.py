"""The streamed host-buffer scan and filter (pip_scan_u64_host,
pip_filter_u64_host — the e2e path of bench.py) with small pipeline chunks,
so the multi-chunk logic runs at test sizes: the carry handed from chunk to
chunk (scan), and the kept prefix of each chunk written back behind the
upload front in order (filter, strong.py:317-327's "destination precedes
source").  Each case runs in a subprocess because the chunk size is read
once per process (PIP_HOST_CHUNK_LOG2 / PIP_HOST_NBUF).

Reference: strong.scan (strong.py:151-166), strong.filter_kway
(strong.py:283-349); oracle: baselines.py:26-41 (oracle/pip_oracle.c).
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

_SUB = r"""
import sys, operator, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2103_01216_b200 as pip
from oracle import oracle
rng = np.random.default_rng(7)
sizes = [1, 2, 65_535, 65_536, 65_537, 131_072, 200_003, 1_000_003, 3 * 65_536 + 5]
for n in sizes:
    for hi in (1 << 20, None):
        x = rng.integers(0, hi or (1 << 63), size=n, dtype=np.uint64) if hi else \
            rng.integers(0, 1 << 64, size=n, dtype=np.uint64)
        # scan: add (inclusive / exclusive), max, min, xor with identities
        for op, ident, name in ((None, 0, None), (max, 5, "max"), (min, 2**64 - 1, "min"),
                                (operator.xor, 0, "xor")):
            a = x.copy()
            r = pip.strong.scan(a, op=op, identity=ident)
            want, tot = oracle.seq_scan(x, op=name, init=(0 if op is None else ident))
            assert np.array_equal(a, want), ("scan", n, name)
            a = x.copy()
            r = pip.strong.scan_inclusive(a, op=op, identity=ident)
            want, tot = oracle.seq_scan(x, op=name, init=(0 if op is None else ident), inclusive=True)
            assert np.array_equal(a, want), ("scan_inclusive", n, name)
        for p in (pip.pred.mod_eq(3, 0), pip.pred.even(), pip.pred.lt(1 << 62), pip.pred.always(),
                  ~pip.pred.always()):
            a = x.copy()
            m = pip.strong.filter_kway(a, p)
            want = oracle.seq_filter(x, p)
            assert m == len(want) and np.array_equal(a[:m], want), ("filter", n, p)
print("ok")
"""


@pytest.mark.parametrize("env", [{"PIP_HOST_CHUNK_LOG2": "16"},
                                 {"PIP_HOST_CHUNK_LOG2": "16", "PIP_HOST_NBUF": "2"},
                                 {"PIP_HOST_CHUNK_LOG2": "17", "PIP_HOST_NBUF": "3"}])
def test_host_scan_filter_small_chunks(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", _SUB, str(ROOT)], env=e, capture_output=True,
                       text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-3000:]
