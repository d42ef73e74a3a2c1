"""The C ABI exactly as include/pip.h documents it (pointer kinds, status
words), called through ctypes the way a non-Python binder would, plus the
stall-reporting path (PIP_ERR_STALLED must surface, never a silent success).

Reference interfaces: strong.scan / filter_kway (strong.py:151-166,
:283-349), relaxed.random_permutation (relaxed.py:220-251), RoundStats
(detres.py:222-230).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys
import textwrap
from pathlib import Path

import numpy as np
import pytest

from conftest import rand_words

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    from paper_2103_01216_b200 import _lib

    return _lib.load()


def _torch_dev(a: np.ndarray):
    import torch

    return torch.from_numpy(a.view(np.int64).copy()).cuda()


def test_scan_filter_device_pointer_kinds(lib, orc):
    """pip_scan_u64 / pip_filter_u64: device array, device total / count,
    device scratch, status via pip_scratch_status."""
    import torch

    from paper_2103_01216_b200 import _lib

    x = rand_words(11, 1_000_003, 1 << 20)
    t = _torch_dev(x)
    scratch = torch.zeros(lib.pip_scratch_bytes(0), dtype=torch.uint8, device="cuda")
    tot = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert lib.pip_scan_u64(t.data_ptr(), len(x), 0, 0, 1, tot.data_ptr(), scratch.data_ptr(),
                            scratch.numel(), st) == 0
    assert lib.pip_scratch_status(scratch.data_ptr(), st) == 0
    want, total = orc.seq_scan(x, inclusive=True)
    assert np.array_equal(t.cpu().numpy().view(np.uint64), want)
    assert int(tot.item()) & ((1 << 64) - 1) == total

    y = rand_words(12, 777_777)
    t = _torch_dev(y)
    m = torch.zeros(1, dtype=torch.int64, device="cuda")
    p = _lib.PipPred(_lib.PRED_MOD_EQ, 0, 3, 0)
    assert lib.pip_filter_u64(t.data_ptr(), len(y), C.byref(p), m.data_ptr(), scratch.data_ptr(),
                              scratch.numel(), st) == 0
    assert lib.pip_scratch_status(scratch.data_ptr(), st) == 0
    kept = y[y % np.uint64(3) == 0]
    assert int(m.item()) == len(kept)
    assert np.array_equal(t.cpu().numpy().view(np.uint64)[: len(kept)], kept)
    # the scratch is too small -> OOM, nothing queued
    assert lib.pip_scan_u64(t.data_ptr(), len(y), 0, 0, 1, tot.data_ptr(), scratch.data_ptr(),
                            16, st) == _lib.PIP_ERR_OOM


def test_rp_device_pointer_kinds(lib, orc):
    """pip_random_permutation_u64: a, h, trace on the DEVICE;
    committed_per_round on the HOST (pip.h); stats on the host."""
    import torch

    from paper_2103_01216_b200 import _lib
    from paper_2103_01216_b200.relaxed import make_swap_sequence
    from paper_2103_01216_b200.runtime import EpsilonConfig, Rng

    n = 300_000
    h = make_swap_sequence(n, Rng(5))
    b = EpsilonConfig(0.5).prefix_words(n)
    a = torch.arange(n, dtype=torch.int64, device="cuda")
    hd = _torch_dev(h)
    nonself = int(np.count_nonzero(h != np.arange(n, dtype=np.uint64)))
    trace = torch.zeros(nonself, dtype=torch.int64, device="cuda")
    cap = 4096
    committed = np.zeros(cap, dtype=np.uint64)  # HOST array
    ws = torch.zeros(lib.pip_rp_workspace_bytes(n, b, 3), dtype=torch.uint8, device="cuda")
    stats = _lib.PipRpStats()
    st = torch.cuda.current_stream().cuda_stream
    rc = lib.pip_random_permutation_u64(a.data_ptr(), hd.data_ptr(), n, b, 3, 0,
                                        committed.ctypes.data, cap, trace.data_ptr(), ws.data_ptr(),
                                        ws.numel(), C.byref(stats), st)
    assert rc == 0
    ref = np.arange(n, dtype=np.uint64)
    info = orc.ref_random_permutation(ref, h, b)
    assert np.array_equal(a.cpu().numpy().view(np.uint64), ref)
    assert stats.rounds == info["rounds"]
    assert committed[: stats.rounds].tolist() == info["committed_per_round"]
    assert stats.total_committed == nonself == int(committed.sum())
    # the trace holds every non-self iterate exactly once
    tr = np.sort(trace.cpu().numpy().view(np.uint64))
    assert np.array_equal(tr, np.flatnonzero(h != np.arange(n, dtype=np.uint64)).astype(np.uint64))


def _run_injected(code: str) -> subprocess.CompletedProcess:
    env = dict(os.environ, PIP_INJECT_STALL="1", PYTHONPATH=str(ROOT))
    return subprocess.run([sys.executable, "-c", textwrap.dedent(code)], env=env, cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


def test_injected_stall_raises_on_device_and_host_paths():
    """A raised stall flag must come back as PIP_ERR_STALLED from every
    look-back op: device scan / filter / reduce through the Python layer, and
    the *_host entry points (each chunk's launch must not clear it)."""
    r = _run_injected("""
        import numpy as np, torch, ctypes as C
        import paper_2103_01216_b200 as pip
        from paper_2103_01216_b200 import _lib
        x = np.arange(3_000_001, dtype=np.uint64)
        hits = []
        for name, fn in [
            ("scan", lambda: pip.strong.scan_inclusive(torch.from_numpy(x.view(np.int64).copy()).cuda())),
            ("filter", lambda: pip.strong.filter_kway(torch.from_numpy(x.view(np.int64).copy()).cuda(), pip.pred.even())),
            ("reduce", lambda: pip.strong.reduce(torch.from_numpy(x.view(np.int64).copy()).cuda())),
            ("scan_host", lambda: pip.strong.scan_inclusive(x.copy())),
            ("filter_host", lambda: pip.strong.filter_kway(x.copy(), pip.pred.even())),
        ]:
            try:
                fn()
                hits.append((name, "ok"))
            except _lib.PipError as e:
                hits.append((name, e.status))
        print(hits)
        assert all(s == _lib.PIP_ERR_STALLED for _, s in hits), hits
        print("INJECTED_OK")
    """)
    assert "INJECTED_OK" in r.stdout, r.stdout + r.stderr


def test_no_stall_without_injection():
    """The same calls succeed when nothing is injected (the flag is cleared
    per public call, so an earlier stall never leaks into a later call)."""
    import torch

    import paper_2103_01216_b200 as pip

    x = np.arange(3_000_001, dtype=np.uint64)
    r = pip.strong.scan_inclusive(torch.from_numpy(x.view(np.int64).copy()).cuda())
    assert r.total == int(x.sum())
    y = x.copy()
    assert pip.strong.filter_kway(y, pip.pred.even()) == (len(x) + 1) // 2
