"""The C ABI's multi-GPU entry points (include/pip.h: pip_scan_u64_sharded,
pip_filter_u64_sharded, pip_filter_shard_plan; csrc/sharded.cu).

CPU: the C plan equals distributed.filter_plan (the plan the gloo tests of
test_distributed.py run at world 2/3/4) on random counts, and applying it to
numpy shards — sends first, then the local shift, then the receives — gives
the sequential filter's packed prefix.
GPU: the entry points on a real NCCL communicator of one rank (this pool has
one GPU per box): allgather, carry kernel and scan / filter through NCCL,
checked against the C oracle."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_2103_01216_b200 import _lib
from paper_2103_01216_b200 import distributed as D
from paper_2103_01216_b200 import pred as P


def c_plan(lib, counts, world, rank, n):
    cn = (C.c_uint64 * world)(*counts)
    down = (_lib.PipShardPiece * max(world, 1))()
    up = (_lib.PipShardPiece * max(world, 1))()
    nd, nu = C.c_int(0), C.c_int(0)
    ss, sl = C.c_uint64(0), C.c_uint64(0)
    rc = lib.pip_filter_shard_plan(cn, world, rank, n, down, C.byref(nd), C.byref(ss), C.byref(sl),
                                   up, C.byref(nu))
    assert rc == 0, rc
    return ([(down[k].peer, down[k].local_offset, down[k].length) for k in range(nd.value)],
            (ss.value, sl.value),
            [(up[k].peer, up[k].local_offset, up[k].length) for k in range(nu.value)])


def test_plan_equals_python_plan():
    lib = _lib.load()
    rng = np.random.default_rng(11)
    for world in (1, 2, 3, 4, 5, 8):
        for n in (0, 1, 7, world, 1000, 12345):
            for _ in range(6):
                sizes = [D.shard_bounds(n, world, r) for r in range(world)]
                counts = [int(rng.integers(0, hi - lo + 1)) for lo, hi in sizes]
                for r in range(world):
                    down, stay, up = D.filter_plan(counts, n, world, r)
                    cd, cs, cu = c_plan(lib, counts, world, r, n)
                    assert cd == [(e, a, b - a) for e, a, b, _ in down]
                    assert cs == (stay[0], stay[1]) or (stay[1] == 0 and cs[1] == 0)
                    assert cu == [(s, d, ln) for s, d, ln in up]


def test_plan_applied_packs_the_global_prefix():
    """Run the C plan on numpy shards with the order the entry point uses."""
    lib = _lib.load()
    rng = np.random.default_rng(5)
    for world, n in ((2, 1001), (3, 5000), (4, 4096), (8, 777)):
        x = rng.integers(0, 1 << 63, size=n, dtype=np.uint64)
        keep = (x % np.uint64(3)) == 0
        shards, counts = [], []
        for r in range(world):
            lo, hi = D.shard_bounds(n, world, r)
            s = x[lo:hi].copy()
            k = s[keep[lo:hi]]
            s[: len(k)] = k
            shards.append(s)
            counts.append(len(k))
        plans = [c_plan(lib, counts, world, r, n) for r in range(world)]
        # 1. sends leave from the untouched arrays
        mail = {}
        for r, (down, _, _) in enumerate(plans):
            for peer, off, ln in down:
                mail.setdefault((r, peer), []).append(shards[r][off:off + ln].copy())
        # 2. local shifts
        for r, (_, (ss, sl), _) in enumerate(plans):
            if sl and ss:
                shards[r][:sl] = shards[r][ss:ss + sl].copy()
        # 3. receives, in plan order per source
        for r, (_, _, up) in enumerate(plans):
            for peer, off, ln in up:
                piece = mail[(peer, r)].pop(0)
                assert len(piece) == ln
                shards[r][off:off + ln] = piece
        assert all(not v for v in mail.values())
        got = np.concatenate(shards)
        m = int(keep.sum())
        assert sum(counts) == m and np.array_equal(got[:m], x[keep])


def test_plan_rejects_bad_arguments():
    lib = _lib.load()
    nd, nu = C.c_int(0), C.c_int(0)
    ss, sl = C.c_uint64(0), C.c_uint64(0)
    down = (_lib.PipShardPiece * 4)()
    cn = (C.c_uint64 * 2)(600, 0)  # more kept words than the shard holds
    assert lib.pip_filter_shard_plan(cn, 2, 0, 1000, down, C.byref(nd), C.byref(ss), C.byref(sl),
                                     down, C.byref(nu)) == _lib.PIP_ERR_INVALID_ARG
    assert lib.pip_filter_shard_plan(cn, 2, 2, 1000, down, C.byref(nd), C.byref(ss), C.byref(sl),
                                     down, C.byref(nu)) == _lib.PIP_ERR_INVALID_ARG
    assert lib.pip_sharded_workspace_bytes(8) == 80 and lib.pip_sharded_workspace_bytes(0) == 0


# ---------------------------------------------------------------------------
# GPU: a real NCCL communicator of one rank

class _NcclId(C.Structure):
    _fields_ = [("internal", C.c_char * 128)]


def _nccl_comm_world1():
    import torch  # noqa: F401  (loads the bundled libnccl)

    nccl = C.CDLL("libnccl.so.2")
    uid = _NcclId()
    nccl.ncclGetUniqueId.argtypes = [C.POINTER(_NcclId)]
    assert nccl.ncclGetUniqueId(C.byref(uid)) == 0
    comm = C.c_void_p()
    nccl.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, _NcclId, C.c_int]
    assert nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0) == 0
    nccl.ncclCommDestroy.argtypes = [C.c_void_p]
    return nccl, comm


@pytest.mark.gpu
def test_sharded_entry_points_on_nccl_world1():
    import torch

    import paper_2103_01216_b200 as pip
    from oracle import oracle

    lib = _lib.load()
    assert lib.pip_nccl_available() == 1
    torch.cuda.set_device(0)
    nccl, comm = _nccl_comm_world1()
    try:
        st = torch.cuda.current_stream().cuda_stream
        sp, sb = pip.runtime.scratch_for(0, st)
        wsb = lib.pip_sharded_workspace_bytes(1)
        ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
        rng = np.random.default_rng(3)
        for n in (0, 1, 100_003, 3_000_001):
            for op, init, inclusive in ((0, 0, 1), (0, 0, 0), (1, 7, 1), (2, (1 << 64) - 1, 0), (3, 0, 1)):
                x = rng.integers(0, 1 << 20, size=n, dtype=np.uint64)
                t = torch.from_numpy(x.view(np.int64).copy()).cuda()
                tot = torch.zeros(1, dtype=torch.int64, device="cuda")
                rc = lib.pip_scan_u64_sharded(t.data_ptr(), n, op, init, inclusive, comm, 0, 1,
                                              ws.data_ptr(), wsb, tot.data_ptr(), sp, sb, st)
                assert rc == 0, rc
                assert lib.pip_scratch_status(sp, st) == 0
                ref = torch.from_numpy(x.view(np.int64).copy()).cuda()
                tot2 = torch.zeros(1, dtype=torch.int64, device="cuda")
                assert lib.pip_scan_u64(ref.data_ptr(), n, op, init, inclusive, tot2.data_ptr(), sp, sb, st) == 0
                torch.cuda.synchronize()
                assert torch.equal(t, ref)
                if n:
                    assert int(tot.item()) == int(tot2.item())
                if op == 0 and n:
                    want, total = oracle.seq_scan(x, inclusive=bool(inclusive))
                    assert np.array_equal(t.cpu().numpy().view(np.uint64), want)
                    assert int(tot.cpu().numpy().view(np.uint64)[0]) == total
            x = rng.integers(0, 1 << 63, size=n, dtype=np.uint64)
            t = torch.from_numpy(x.view(np.int64).copy()).cuda()
            p = P.mod_eq(3, 0)
            desc = p.descriptor()
            m, ln = C.c_uint64(0), C.c_uint64(0)
            rc = lib.pip_filter_u64_sharded(t.data_ptr(), n, n, C.byref(desc), comm, 0, 1, ws.data_ptr(),
                                            wsb, C.byref(m), C.byref(ln), sp, sb, st)
            assert rc == 0, rc
            want = oracle.seq_filter(x, p)
            assert m.value == len(want) == ln.value
            assert np.array_equal(t.cpu().numpy().view(np.uint64)[: m.value], want)
        # argument checks: wrong rank / world for this communicator, short workspace
        t = torch.zeros(16, dtype=torch.int64, device="cuda")
        assert lib.pip_scan_u64_sharded(t.data_ptr(), 16, 0, 0, 1, comm, 1, 2, ws.data_ptr(), 8 * 4, None,
                                        sp, sb, st) == _lib.PIP_ERR_INVALID_ARG
        assert lib.pip_scan_u64_sharded(t.data_ptr(), 16, 0, 0, 1, comm, 0, 1, ws.data_ptr(), 8, None,
                                        sp, sb, st) == _lib.PIP_ERR_OOM
        assert lib.pip_scan_u64_sharded(t.data_ptr(), 16, 0, 0, 1, None, 0, 1, ws.data_ptr(), wsb, None,
                                        sp, sb, st) == _lib.PIP_ERR_INVALID_ARG
    finally:
        torch.cuda.synchronize()
        nccl.ncclCommDestroy(comm)
