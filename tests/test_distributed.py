"""Multi-rank plan of the sharded scan / filter / merge (paper_2103_01216_b200
/distributed.py) on CPU: gloo, world sizes 2, 3 and 4, with the C oracle
standing in for the per-rank CUDA kernels (the device kernels themselves are
covered by the -m gpu tests, and test_sharded_*_cuda_gloo runs the same plans
with the libpip kernels on one GPU).  Checks: the global result equals the
sequential oracle; the filter and merge stay in place (no rank allocates
more than the bounded exchange ring)."""
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

    def move(self, t, dst, src, length):
        t[dst:dst + length] = t[src:src + length].clone()

    def reverse(self, t):
        t.copy_(t.flip(0))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q, cuda=False, backend="gloo"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if backend == "nccl":
        torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        if cuda:
            torch.cuda.set_device(0)
            ops = D.CudaOps()
        else:
            ops = OracleOps()
        res = []
        for case in cases:
            name, n = case[0], case[1]
            g = _global(case)
            lo, hi = D.shard_bounds(n, world, rank)
            local = torch.from_numpy(g[lo:hi].view(np.int64).copy())
            if cuda:
                local = local.cuda()
            ptr = local.data_ptr()
            if name == "scan":
                r0 = D.sharded_scan(local, ops, inclusive=True)
            elif name == "filter":
                r0 = D.sharded_filter(local, n, _PREDS[case[3]], ops)
            else:
                D.sharded_merge(local, n, _split(case), ops, wave_words=case[4])
                r0 = 0
            assert local.data_ptr() == ptr  # in place: the caller's buffer
            res.append((r0, local.cpu().numpy().view(np.uint64).copy()))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


_PREDS = {"mod3": P.mod_eq(3, 0), "all": P.always(), "none": ~P.always(), "lt": P.lt(1 << 61)}


def _split(case):
    name, n, seed, kind, wave = case
    return {"half": n // 2 + 3, "zero": 0, "all": n, "small": 5}[kind]


def _run(world, cases, cuda=False, backend="gloo"):
    """Run every case in one process group; returns, per case, the ranks'
    (result, final shard) in rank order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q, cuda, backend))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda x: x[0])
    return [[o[1][k] for o in out] for k in range(len(cases))]


def _global(case):
    name, n, seed = case[0], case[1], case[2]
    rng = np.random.default_rng(seed)
    if name == "scan":
        return rng.integers(0, 1 << 64, size=n, dtype=np.uint64)
    if name == "filter":
        return rng.integers(0, 1 << 63, size=n, dtype=np.uint64)
    na = _split(case)
    hi = {1: 97, 2: 1 << 64, 3: 1}.get(seed % 4, 97)
    a = np.sort(rng.integers(0, hi, size=na, dtype=np.uint64))
    b = np.sort(rng.integers(0, hi, size=n - na, dtype=np.uint64))
    if seed % 4 == 0:  # disjoint: every A word above every B word
        a = a + np.uint64(1000)
    return np.concatenate([a, b])


MERGE_CASES = [(1, "half", 1 << 22), (1, "half", 7), (2, "half", 64), (3, "half", 33),
               (4, "half", 100), (4, "small", 13), (5, "zero", 50), (5, "all", 50)]


def _check(case, per_rank):
    g = _global(case)
    got = np.concatenate([r[1] for r in per_rank])
    if case[0] == "scan":
        want = np.cumsum(g, dtype=np.uint64)
        assert np.array_equal(got, want), case
        assert all(r[0] == int(want[-1]) for r in per_rank), case
    elif case[0] == "filter":
        want = g[_PREDS[case[3]](g)]
        m = per_rank[0][0]
        assert all(r[0] == m for r in per_rank) and m == len(want), case
        assert np.array_equal(got[:m], want), case
    else:
        assert np.array_equal(got, np.sort(g)), case


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_gloo(world):
    """scan, filter (4 predicates: ~1/3, all, none, most kept) and merge (8
    run shapes: duplicates, full-range words, one value, disjoint runs, tiny
    / empty / whole-array first run, exchange rings of 7 to 2^22 words)."""
    cases = [("scan", 10_007, 1)]
    cases += [("filter", 9_001, 2, k) for k in ("mod3", "all", "none", "lt")]
    cases += [("merge", 8_000 + seed, seed, kind, wave) for seed, kind, wave in MERGE_CASES]
    for case, per_rank in zip(cases, _run(world, cases)):
        _check(case, per_rank)


def test_merge_interleave_plan_levels():
    # 8 shards: 3 levels, each rotation inside its group's range
    S, n = 100, 800
    cr = [0, 10, 60, 100, 180, 250, 300, 390, 400]
    q = [d * S for d in range(9)]
    levels = D.merge_interleave_plan(cr, q, 8)
    assert [len(lv) for lv in levels] == [1, 2, 4]
    x, y, z = levels[0][0]
    assert (x, y, z) == (cr[4], cr[8], cr[8] + (4 * S - cr[4]))


def test_filter_plan_destinations_precede_sources():
    counts, n, world = [3, 50, 0, 100, 7], 500, 5
    offs = np.concatenate([[0], np.cumsum(counts)])
    for r in range(world):
        down, (s0, slen), up = D.filter_plan(counts, n, world, r)
        lo, _ = D.shard_bounds(n, world, r)
        for e, a, b, d in down:
            assert e < r and b - a > 0
        assert s0 + slen == counts[r] and (slen == 0 or offs[r] + s0 == lo)
        for s, d, ln in up:
            assert s > r and d >= slen


@pytest.mark.gpu
def test_sharded_cuda_gloo():
    """The same plans with the libpip kernels as the local ops, two ranks on
    one GPU (gloo moves the data through the host; the ranks' kernels never
    wait on one another)."""
    cases = [("filter", 300_007, 2, "mod3"), ("scan", 200_003, 1),
             ("merge", 400_009, 1, "half", 1 << 12), ("merge", 300_001, 4, "half", 1000)]
    for case, per_rank in zip(cases, _run(2, cases, cuda=True)):
        _check(case, per_rank)


@pytest.mark.gpu
def test_sharded_cuda_nccl_world1():
    """The sharded plans over the NCCL backend itself (the backend the SCALE
    run uses), as far as one GPU allows: a process group of one rank, so
    every collective (all_gather of totals / counts, the co-rank search's
    all_reduce on int64 words) really goes through NCCL on device buffers."""
    cases = [("filter", 300_007, 2, "mod3"), ("scan", 200_003, 1),
             ("merge", 400_009, 1, "half", 1 << 12), ("merge", 100_001, 4, "small", 1000)]
    for case, per_rank in zip(cases, _run(1, cases, cuda=True, backend="nccl")):
        _check(case, per_rank)


@pytest.mark.gpu
@pytest.mark.parametrize("op", ["scan", "filter", "merge"])
def test_bench_sharded_paths_one_gpu(op):
    """bench.py's N>1 paths (the SCALE run's code) end to end with two ranks
    on one GPU over gloo (PIP_ONE_GPU=1): parity checks inside the bench
    pass and rank 0 prints one JSON line.  Functional only: numbers of such
    a run are not bench values."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, PIP_ONE_GPU="1", PIP_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", "--op", op, "--log2n", "22", "--steps", "2", "--warmup", "1",
           "--no-e2e", "--no-cpu"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["n"] == 1 << 22
