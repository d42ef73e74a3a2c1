"""Multi-rank plan of the sharded scan / filter / merge (paper_2103_01216_b200
/distributed.py) on CPU: gloo, world sizes 2 and 3, with the C oracle standing
in for the per-rank CUDA kernels (the device kernels themselves are covered by
the -m gpu tests)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_01216_b200 import distributed as D
from paper_2103_01216_b200 import pred as P

M64 = (1 << 64) - 1


class OracleOps(D.LocalOps):
    """numpy/C-oracle local ops on CPU int64 tensors (test stand-in only)."""

    device = torch.device("cpu")

    def __init__(self):
        from oracle import oracle

        self.o = oracle

    @staticmethod
    def _u(t):
        return t.numpy().view(np.uint64)

    def reduce(self, t):
        s = int(self._u(t).sum(dtype=np.uint64))
        return torch.tensor([np.uint64(s).view(np.int64)], dtype=torch.int64)

    def scan_carry(self, t, carry, inclusive):
        c = int(carry.numpy().view(np.uint64)[0])
        out, _ = self.o.seq_scan(self._u(t), inclusive=inclusive, init=c)
        t.numpy()[:] = out.view(np.int64)

    def filter(self, t, pred):
        kept = self.o.seq_filter(self._u(t), pred)
        t.numpy()[: len(kept)] = kept.view(np.int64)
        return len(kept)

    def merge(self, t, split):
        u = self._u(t)
        out = self.o.seq_merge(u[:split].copy(), u[split:].copy())
        t.numpy()[:] = out.view(np.int64)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ops = OracleOps()
        name, n, seed = case
        rng = np.random.default_rng(seed)
        if name == "scan":
            g = rng.integers(0, 1 << 64, size=n, dtype=np.uint64)
        elif name == "filter":
            g = rng.integers(0, 1 << 63, size=n, dtype=np.uint64)
        else:
            na = n // 2 + 3
            g = np.concatenate([np.sort(rng.integers(0, 97, size=na, dtype=np.uint64)),
                                np.sort(rng.integers(0, 97, size=n - na, dtype=np.uint64))])
        lo, hi = D.shard_bounds(n, world, rank)
        local = torch.from_numpy(g[lo:hi].view(np.int64).copy())
        if name == "scan":
            tot = D.sharded_scan(local, ops, inclusive=True)
            res = (tot, local.numpy().view(np.uint64).copy())
        elif name == "filter":
            m = D.sharded_filter(local, n, P.mod_eq(3, 0), ops)
            res = (m, local.numpy().view(np.uint64).copy())
        else:
            D.sharded_merge(local, n, n // 2 + 3, ops)
            res = (0, local.numpy().view(np.uint64).copy())
        q.put((rank, res[0], res[1]))
    finally:
        dist.destroy_process_group()


def _run(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda x: x[0])
    return out


def _global(case):
    name, n, seed = case
    rng = np.random.default_rng(seed)
    if name == "scan":
        return rng.integers(0, 1 << 64, size=n, dtype=np.uint64)
    if name == "filter":
        return rng.integers(0, 1 << 63, size=n, dtype=np.uint64)
    na = n // 2 + 3
    return np.concatenate([np.sort(rng.integers(0, 97, size=na, dtype=np.uint64)),
                           np.sort(rng.integers(0, 97, size=n - na, dtype=np.uint64))])


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_scan_gloo(world):
    case = ("scan", 10_007, 1)
    out = _run(world, case)
    g = _global(case)
    want = np.cumsum(g, dtype=np.uint64)
    got = np.concatenate([o[2] for o in out])
    assert np.array_equal(got, want)
    assert all(o[1] == int(want[-1]) for o in out)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_filter_gloo(world):
    case = ("filter", 9_001, 2)
    out = _run(world, case)
    g = _global(case)
    want = g[(g % np.uint64(3)) == 0]
    m = out[0][1]
    assert all(o[1] == m for o in out) and m == len(want)
    got = np.concatenate([o[2] for o in out])[:m]
    assert np.array_equal(got, want)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_merge_gloo(world):
    case = ("merge", 8_000, 3)
    out = _run(world, case)
    g = _global(case)
    got = np.concatenate([o[2] for o in out])
    assert np.array_equal(got, np.sort(g))
