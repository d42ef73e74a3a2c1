"""GPU parity of the host-buffer random permutation (pip_random_permutation_u64_host,
the C-ABI call bench.py's e2e leg makes): output against the sequential Knuth
swap order (relaxed.py:220-251 / the C oracle) and round statistics against
the device entry point.  Above 2^23 words the final suffix is copied back
while the rounds run (progress word after every round); the overlap is
checked with pageable and pinned host arrays, several budgets and variants,
and against PIP_RP_HOST_OVERLAP=0 in a subprocess."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
VARIANT = {"naive": 0, "flat": 1, "oneres": 2, "final": 3}


def run_host(a: np.ndarray, h: np.ndarray, prefix: int, variant: str):
    from paper_2103_01216_b200 import _lib

    lib = _lib.load()
    st = _lib.PipRpStats()
    rc = lib.pip_random_permutation_u64_host(a.ctypes.data, h.ctypes.data, len(a), prefix,
                                             VARIANT[variant], C.byref(st), 0)
    assert rc == 0, lib.pip_status_string(rc)
    return st


@pytest.mark.parametrize("n,prefix,variant", [
    ((1 << 23) + 4099, 1 << 18, "final"),
    ((1 << 24) + 3, None, "final"),
    ((1 << 23) + 1, 1 << 17, "oneres"),
    ((1 << 22) + 5, 1 << 16, "final"),  # below the overlap threshold
])
def test_rp_host_matches_knuth_and_device(orc, n, prefix, variant):
    import torch

    import paper_2103_01216_b200 as pip

    if prefix is None:
        prefix = pip.EpsilonConfig(0.5).prefix_words(n)
    h = pip.relaxed.make_swap_sequence(n, pip.Rng(7))
    want = np.arange(n, dtype=np.uint64)
    orc.seq_knuth_shuffle(want, h)
    a = np.arange(n, dtype=np.uint64)
    st = run_host(a, h, prefix, variant)
    assert np.array_equal(a, want)
    # the same call on device buffers: identical round structure
    da = torch.arange(n, dtype=torch.int64, device="cuda")
    dh = torch.from_numpy(h.view(np.int64)).cuda()
    bud = pip.EpsilonConfig(0.5, prefix / n)
    sd = pip.relaxed.random_permutation(da, dh, variant=variant, budget=bud)
    if bud.prefix_words(n) == prefix:
        assert st.rounds == sd.rounds and st.total_committed == sd.total_committed
    assert np.array_equal(da.cpu().numpy().view(np.uint64), want)


def test_rp_host_pinned_and_permuted_input(orc):
    import torch

    import paper_2103_01216_b200 as pip

    n = (1 << 23) + 77
    h = pip.relaxed.make_swap_sequence(n, pip.Rng(11))
    x = np.random.default_rng(5).integers(0, 1 << 64, n, dtype=np.uint64)
    want = x.copy()
    orc.seq_knuth_shuffle(want, h)
    t = torch.from_numpy(x.view(np.int64).copy()).pin_memory()
    th = torch.from_numpy(h.view(np.int64).copy()).pin_memory()
    from paper_2103_01216_b200 import _lib

    st = _lib.PipRpStats()
    rc = _lib.load().pip_random_permutation_u64_host(t.data_ptr(), th.data_ptr(), n, 1 << 17, 3,
                                                     C.byref(st), 0)
    assert rc == 0
    assert np.array_equal(t.numpy().view(np.uint64), want)


_SUB = r"""
import sys, ctypes as C, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2103_01216_b200 as pip
from paper_2103_01216_b200 import _lib
n = (1 << 23) + 999
h = pip.relaxed.make_swap_sequence(n, pip.Rng(9))
a = np.arange(n, dtype=np.uint64)
st = _lib.PipRpStats()
assert _lib.load().pip_random_permutation_u64_host(a.ctypes.data, h.ctypes.data, n, 1 << 18, 3,
                                                   C.byref(st), 0) == 0
np.save(sys.argv[2], a)
print(st.rounds)
"""


def test_rp_host_overlap_off_identical(tmp_path):
    outs = []
    for v in ("0", "1"):
        f = tmp_path / f"a{v}.npy"
        r = subprocess.run([sys.executable, "-c", _SUB, str(ROOT), str(f)],
                           env=dict(os.environ, PIP_RP_HOST_OVERLAP=v), capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append((np.load(f), r.stdout.strip()))
    assert np.array_equal(outs[0][0], outs[1][0]) and outs[0][1] == outs[1][1]
