"""pip_move_u64 (the sharded filter's in-place shift and the relaxed
filter's per-round move) and pip_reverse_u64 (the sharded merge's mirror
swaps): memmove semantics on one device array, every overlap shape."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2103_01216_b200 as pip
    from paper_2103_01216_b200 import _lib

    return torch, pip, _lib.load(), _lib


@pytest.mark.parametrize("n,dst,src,length", [
    (100, 0, 1, 99), (100, 0, 50, 50), (100, 10, 60, 30), (10_000, 3, 5, 9_000),
    (3_000_017, 1, 2, 3_000_000), (3_000_017, 0, 1_000_000, 2_000_000),
    (3_000_017, 7, 6_661, 2_993_000), (2_000_000, 5, 6, 1),
    (100, 5, 1, 90), (3_000_017, 2, 1, 3_000_000),            # right moves (rotation)
    (100, 60, 0, 30), (3_000_017, 2_000_000, 0, 1_000_000),   # disjoint
    (50, 3, 3, 40), (50, 0, 10, 0)])
def test_move_matches_memmove(env, n, dst, src, length):
    torch, pip, lib, _lib = env
    x = np.random.default_rng(n + dst + src).integers(0, 1 << 64, size=n, dtype=np.uint64)
    t = torch.from_numpy(x.view(np.int64).copy()).cuda()
    st = torch.cuda.current_stream().cuda_stream
    sp, sb = pip.runtime.scratch_for(0, st)
    _lib.check(lib.pip_move_u64(t.data_ptr(), dst, src, length, sp, sb, st), "move")
    _lib.check_stall(sp, st, "move")
    got = t.cpu().numpy().view(np.uint64)
    want = x.copy()
    want[dst:dst + length] = x[src:src + length]
    # only the destination range is specified (a right move rotates the rest)
    assert np.array_equal(got[dst:dst + length], want[dst:dst + length])
    outside = np.ones(n, dtype=bool)
    outside[min(dst, src):max(dst, src) + length] = False
    assert np.array_equal(got[outside], x[outside])


@pytest.mark.parametrize("n", [0, 1, 2, 3, 1000, 1_000_001])
def test_reverse(env, n):
    torch, pip, lib, _lib = env
    x = np.random.default_rng(n).integers(0, 1 << 64, size=n, dtype=np.uint64)
    t = torch.from_numpy(x.view(np.int64).copy()).cuda()
    if n:
        _lib.check(lib.pip_reverse_u64(t.data_ptr(), n, torch.cuda.current_stream().cuda_stream),
                   "reverse")
    assert np.array_equal(t.cpu().numpy().view(np.uint64), x[::-1])
