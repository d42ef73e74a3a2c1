#!/usr/bin/env python
"""Benchmark of the PIP hot path on B200 (contract: one JSON line on rank 0).

Default workload (N=1): BASELINE.json configs[1] — in-place INCLUSIVE prefix
sum of n = 2^32 int64 words, values Rng(1).words >> 44 (uniform in [0, 2^20)),
resident in HBM.  `--op` selects the other configs for our own measurements:
  scan    configs[1]  inclusive scan, 2^32 words               (default)
  filter  configs[2]  stable filter x % 3 == 0, 2^32 words, values < 2^63
  merge   configs[3]  merge two sorted runs of 2^31 words, values < 2^30
  rp      configs[4]  random permutation, n = 2^30, H = make_swap_sequence
  rp0     configs[0]  random permutation, n = 10^6, H from PCG64(seed)
  partition  SURVEY 8(f) row 3 (not a BASELINE config): unstable in-place
          partition, 2^32 words with the configs[2] inputs and predicate
Multi-GPU (torchrun, WORLD_SIZE = N > 1), strong scaling over 2^32 / N words
per rank: scan (local reduce -> NCCL all_gather of shard totals -> scan with
a device carry-in), filter (local filter -> in-place NCCL P2P moves to the
global packed prefix) and merge (collective co-ranks -> in-place rotations
of shard pieces -> local merge); see paper_2103_01216_b200/distributed.py.  `--impl reference` times the CPU reference
path (the C port of the reference's own algorithm in oracle/) instead.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PAPER_GELEM_S = {  # PAPER.md:1148-1157,1320-1332 (72-core Xeon, Cilk Plus), for context only
    "scan": 2e9 / 0.336, "filter": 2e9 / 0.335, "rp": 1e9 / 3.960, "rp0": 1e7 / 0.0656,
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="pip", choices=["pip", "reference"])
    ap.add_argument("--op", default="scan",
                    choices=["scan", "filter", "merge", "rp", "rp0", "partition"])
    ap.add_argument("--log2n", type=int, default=None, help="override n = 2^k")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--profile", action="store_true",
                    help="single warm launch pair for ncu (no JSON contract)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing

def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist

        # PIP_DIST_BACKEND=gloo + PIP_ONE_GPU=1: every rank on cuda:0 with
        # gloo (functional test of the sharded paths on a one-GPU box; the
        # numbers of such a run are not bench values)
        if os.environ.get("PIP_ONE_GPU") == "1":
            local = 0
        torch.cuda.set_device(local)
        backend = os.environ.get("PIP_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.proc = None
        self.path = tempfile.mktemp(prefix="clk", suffix=".csv")
        try:
            import torch

            uuid = str(torch.cuda.get_device_properties(device).uuid)
            sel = uuid if uuid.startswith("GPU-") else f"GPU-{uuid}"
        except Exception:
            sel = str(device)
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", sel, f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.f, stderr=subprocess.DEVNULL)
            # nvidia-smi takes a moment to start (and may buffer its output):
            # give it time to be sampling before a short timed region begins
            time.sleep(0.6)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no-samples"]}
        # median under load: samples at >= 50% of max (idle gaps excluded)
        hi = [s for s in sm if s >= 0.5 * max(smax)] or sm
        return {"sm_mhz": statistics.median(hi), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# helpers

def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "MEASURED_PEAKS.json (measured copy)"}
    return {"hbm_gbs": 6650.0, "source": "B200_PROFILING.md fallback 6.65 TB/s"}


def ncu_traffic(op: str):
    """DRAM bytes per element of the dominant kernel from the committed ncu
    summary (profiles/ncu_summary.json), or None."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    e = d.get(op)
    if not e:
        return None
    return e.get("dram_bytes_per_elem")


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


class Events:
    def __init__(self, torch):
        self.torch = torch

    def time(self, fn, steps: int, stream):
        torch = self.torch
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1)


# ---------------------------------------------------------------------------
# workloads (pip arm)

def run_scan(args, ws, rank, local, torch, pip, lib):
    n_total = 1 << (args.log2n or 32)
    n = n_total // ws
    lo = rank * n
    dev = local
    st = torch.cuda.current_stream()
    sptr = st.cuda_stream
    a = torch.empty(n, dtype=torch.int64, device=f"cuda:{dev}")
    pip.Rng(args.seed).words_device(lo, lo + n, shift=44, device=dev, out=a)
    torch.cuda.synchronize()
    sp, sb = pip.runtime.scratch_for(dev, sptr)
    tot = torch.zeros(ws + 2, dtype=torch.int64, device=f"cuda:{dev}")
    gathered = torch.zeros(ws, dtype=torch.int64, device=f"cuda:{dev}")
    carry = torch.zeros(1, dtype=torch.int64, device=f"cuda:{dev}")

    if ws == 1:
        def step():
            rc = lib.pip_scan_u64(a.data_ptr(), n, 0, 0, 1, tot.data_ptr(), sp, sb, sptr)
            assert rc == 0, rc
        # scan_ws2_kernel over the whole 6656-word tiles + the register
        # kernel for the ragged tail (csrc/scan.cu launch_scan_ws2)
        launches = 1 + (1 if n % 6656 else 0)
    else:
        import torch.distributed as dist

        nccl = dist.get_backend() == "nccl"

        def step():
            # shard total -> all ranks' totals -> exclusive carry -> scan with carry
            rc = lib.pip_reduce_u64(a.data_ptr(), n, 0, tot.data_ptr(), sp, sb, sptr)
            assert rc == 0, rc
            if nccl:
                dist.all_gather_into_tensor(gathered, tot[:1])
            else:  # gloo (functional one-GPU runs): list form
                parts = list(gathered.split(1))
                dist.all_gather(parts, tot[:1].clone())
            torch.sum(gathered[:rank], dim=0, keepdim=True, out=carry) if rank else carry.zero_()
            rc = lib.pip_scan_u64_carry(a.data_ptr(), n, 0, 0, 1, carry.data_ptr(),
                                        tot[1:].data_ptr(), sp, sb, sptr)
            assert rc == 0, rc
        launches = 2

    # parity of the first (warm-up) step through a size-independent property:
    # the inclusive scan's adjacent differences give back the input, on
    # windows at the start, middle and end of the shard, plus the total
    wins = [(0, 1 << 16), (n // 2 - 4096, n // 2 + 4096), (n - (1 << 16), n)]
    before = [a[s:e].clone() for s, e in wins]
    step()
    torch.cuda.synchronize()
    for (s, e), x in zip(wins, before):
        out = a[s:e]
        assert torch.equal(out[1:] - out[:-1], x[1:]), f"scan parity failed on window {s}"
    if ws == 1:
        assert int(tot[0].item()) == int(a[n - 1].item())
        assert int(a[0].item()) == int(before[0][0].item())
    for _ in range(max(args.warmup - 1, 0)):
        step()
    torch.cuda.synchronize()

    barrier(ws)
    torch.cuda.synchronize()
    clk = ClockSampler(dev)
    ms = Events(torch).time(step, args.steps, st)
    torch.cuda.synchronize()
    barrier(ws)
    clocks = clk.stop()
    ms = max_over_ranks(ms, ws)
    per_step = ms / args.steps
    value = n_total * args.steps / (ms / 1e3)
    # roofline: dominant kernel = scan_kernel; 16 B/elem algorithmic (ws==1)
    algo_bytes = 16 * n if ws == 1 else 24 * n
    pk = peaks()
    achieved = algo_bytes / (per_step / 1e3) / 1e9
    tb = ncu_traffic("scan")
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"],
            "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4),
            "traffic": (tb * n) if tb else None,
            "note": f"{'16' if ws == 1 else '24'} B/word algorithmic (read+write"
                    f"{'' if ws == 1 else ' + shard reduce'}); peak = {pk['source']}; "
                    "kernel time = CUDA-event step time (1 launch/step); the peak is the "
                    "bandwidth a torch copy measured on this pool, not the HBM limit, so a "
                    "short run of this kernel can reach or pass 1.0 of it"}
    extra = {"n_per_rank": n}
    e2e = None
    if not args.no_e2e:
        e2e = e2e_host(lib, "scan", n, args, torch, dev, ws)
    cpu = None
    if ws == 1 and rank == 0 and not args.no_cpu:
        cpu = cpu_baseline("scan", args)
    cfg = {"workload": "inclusive in-place scan, BASELINE configs[1]", "n": n_total,
           "dtype_in": "int64 (uint64 words)", "values": f"Rng({args.seed}).words >> 44, in [0,2^20)",
           "l2": "inputs (32 GiB) larger than L2 (126 MB): no flush needed",
           "parallelism": f"shard{ws}" if ws > 1 else "single-GPU",
           "seed": args.seed}
    return dict(value=value, per_step=per_step, roof=roof, e2e=e2e, cpu=cpu, cfg=cfg,
                clocks=clocks, launches=launches * args.steps, extra=extra)


def regen_timed(step, regen, steps, torch, st, ws: int = 1):
    """Per-step CUDA-event timing for destructive in-place ops: the input is
    regenerated between steps OUTSIDE the timed events (ranks meet at a
    barrier before each timed step)."""
    total = 0.0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for _ in range(steps):
        regen()
        torch.cuda.synchronize()
        barrier(ws)
        e0.record(st)
        step()
        e1.record(st)
        e1.synchronize()
        total += e0.elapsed_time(e1)
    return total


def _windows(n: int, w: int = 1 << 20):
    w = min(w, n)
    mid = max(0, n // 2 - w // 2)
    return sorted({(0, w), (mid, mid + w), (n - w, n)})


def check_filter_windows(a, src, m, pred, lib, desc, sp, sb, sptr, torch):
    """Oracle parity of a filtered array on sampled input windows."""
    from oracle import oracle

    n = src.numel()
    cnt = torch.zeros(1, dtype=torch.int64, device=src.device)
    assert lib.pip_count_u64(src.data_ptr(), n, C.byref(desc), cnt.data_ptr(), sp, sb, sptr) == 0
    assert int(cnt.item()) == m, "filter count parity failed"
    for lo, hi in _windows(n):
        pos = 0
        if lo:
            assert lib.pip_count_u64(src.data_ptr(), lo, C.byref(desc), cnt.data_ptr(), sp, sb,
                                     sptr) == 0
            pos = int(cnt.item())
        kept = oracle.seq_filter(src[lo:hi].cpu().numpy().view(np.uint64), pred)
        got = a[pos:pos + len(kept)].cpu().numpy().view(np.uint64)
        assert np.array_equal(got, kept), f"filter parity failed on input window [{lo}, {hi})"


def merge_coranks(A, B, ranks, torch):
    """Merge-path co-ranks (ties from A, strong.py:474-488) of several output
    ranks at once (vectorised bisection on the device)."""
    na, nb = A.numel(), B.numel()
    r = torch.tensor(ranks, dtype=torch.int64, device=A.device)
    lo = torch.clamp(r - nb, min=0)
    hi = torch.clamp(r, max=na)
    flip = -(1 << 63)
    while bool((lo < hi).any()):
        act = lo < hi
        mid = torch.where(act, (lo + hi) // 2, torch.zeros_like(lo))
        bj = torch.where(act, r - mid - 1, torch.zeros_like(lo))
        go = act & ((B[bj.clamp(0, nb - 1)] ^ flip) >= (A[mid.clamp(0, na - 1)] ^ flip))
        lo = torch.where(go, mid + 1, lo)
        hi = torch.where(act & ~go, mid, hi)
    return lo.tolist()


def check_merge_windows(a, orig, na, torch):
    """Oracle parity of a merged array on sampled output windows."""
    from oracle import oracle

    n = a.numel()
    A, B = orig[:na], orig[na:]
    for r0, r1 in _windows(n):
        i0, i1 = merge_coranks(A, B, [r0, r1], torch)
        want = oracle.seq_merge(A[i0:i1].cpu().numpy().view(np.uint64),
                                B[r0 - i0:r1 - i1].cpu().numpy().view(np.uint64))
        got = a[r0:r1].cpu().numpy().view(np.uint64)
        assert np.array_equal(got, want), f"merge parity failed on output window [{r0}, {r1})"


def _wsum(t, w, torch):
    """sum(t * w) mod 2^64 (int64 wrap-around), as a signed int64 value."""
    v = int((t * w).sum().item()) & ((1 << 64) - 1)
    return v - (1 << 64) if v >> 63 else v


def run_filter_sharded(args, ws, rank, local, torch, pip, lib):
    """configs[2] over ws GPUs (strong scaling): rank r filters its 2^32/ws
    words, then the kept words move in place to the global packed prefix
    (distributed.sharded_filter)."""
    import torch.distributed as dist

    from paper_2103_01216_b200 import distributed as D

    n_total = 1 << (args.log2n or 32)
    lo, hi = D.shard_bounds(n_total, ws, rank)
    n = hi - lo
    dev = local
    st = torch.cuda.current_stream()
    a = torch.empty(n, dtype=torch.int64, device=f"cuda:{dev}")
    rng = pip.Rng(args.seed)
    regen = lambda: rng.words_device(lo, hi, shift=1, device=dev, out=a)  # noqa: E731
    p = pip.pred.mod_eq(3, 0)
    ops = D.CudaOps()
    res = {}

    def step():
        res["m"] = D.sharded_filter(a, n_total, p, ops)

    # parity of the first step by an order-sensitive checksum: every kept
    # word x with global kept rank k contributes x * (k + 1) (mod 2^64);
    # computed from the input shards and from the packed output
    regen()
    keep = (a % 3) == 0
    c = int(keep.sum().item())
    cnt = torch.tensor([c], dtype=torch.int64, device=a.device)
    allc = [torch.zeros_like(cnt) for _ in range(ws)]
    dist.all_gather(allc, cnt)
    off = sum(int(x.item()) for x in allc[:rank])
    kept = a[keep]
    w_in = torch.tensor([_wsum(kept, torch.arange(off + 1, off + 1 + c, device=a.device), torch),
                         _wsum(kept, 1, torch)], dtype=torch.int64, device=a.device)
    del kept, keep
    step()
    torch.cuda.synchronize()
    m = res["m"]
    assert m == sum(int(x.item()) for x in allc), "sharded filter count"
    top = max(0, min(hi, m) - lo)
    out = a[:top]
    w_out = torch.tensor([_wsum(out, torch.arange(lo + 1, lo + 1 + top, device=a.device), torch),
                          _wsum(out, 1, torch)], dtype=torch.int64, device=a.device)
    both = torch.stack([w_in, w_out])
    dist.all_reduce(both)
    assert torch.equal(both[0], both[1]), "sharded filter checksum parity failed"
    for _ in range(max(args.warmup - 1, 0)):
        regen()
        step()
    torch.cuda.synchronize()
    barrier(ws)
    clk = ClockSampler(dev)
    ms = regen_timed(step, regen, args.steps, torch, st, ws=ws)
    clocks = clk.stop()
    ms = max_over_ranks(ms, ws)
    per_step = ms / args.steps
    value = n_total * args.steps / (ms / 1e3)
    pk = peaks()
    algo = 8 * n + 8 * (m / ws)  # per GPU: read my shard once, write my share of the prefix
    achieved = algo / (per_step / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": None,
            "note": "per GPU: 8 B/word of its shard + 8 B per word of its share of the packed "
                    "prefix; the step also moves the kept words across GPUs (NCCL P2P)"}
    cfg = {"workload": "stable in-place filter x % 3 == 0, BASELINE configs[2]", "n": n_total,
           "n_per_rank": n, "values": f"Rng({args.seed}).words >> 1, in [0,2^63)", "kept": m,
           "l2": "inputs larger than L2; input regenerated between steps (untimed)",
           "parallelism": f"shard{ws}: local filter + in-place P2P moves to the global prefix",
           "check": "order-sensitive checksum of the packed prefix vs the inputs",
           "seed": args.seed}
    return dict(value=value, per_step=per_step, roof=roof, e2e=None, cpu=None, cfg=cfg,
                clocks=clocks, launches=2 * args.steps, extra={})


def run_merge_sharded(args, ws, rank, local, torch, pip, lib):
    """configs[3] over ws GPUs (strong scaling): each rank holds 2^32/ws words
    of the two sorted runs; co-ranks by a collective 4096-ary search, the
    shard interleave by in-place rotations (P2P mirror swaps), local merge
    (distributed.sharded_merge)."""
    import torch.distributed as dist

    from paper_2103_01216_b200 import distributed as D

    n_total = 1 << (args.log2n or 32)
    na = n_total // 2
    lo, hi = D.shard_bounds(n_total, ws, rank)
    n = hi - lo
    dev = local
    st = torch.cuda.current_stream()
    # every rank builds the same global sorted runs (same generator and sort
    # as one GPU), keeps its shard as the pristine input, and checks its
    # output window against the oracle from the global runs
    g = torch.empty(n_total, dtype=torch.int64, device=f"cuda:{dev}")
    pip.Rng(args.seed).words_device(0, n_total, shift=34, device=dev, out=g)
    sort_run(g[:na], torch, pip)
    sort_run(g[na:], torch, pip)
    orig = g[lo:hi].clone()
    A, B = g[:na], g[na:]
    a = torch.empty(n, dtype=torch.int64, device=f"cuda:{dev}")
    regen = lambda: a.copy_(orig)  # noqa: E731
    ops = D.CudaOps()

    def step():
        D.sharded_merge(a, n_total, na, ops)

    regen()
    step()
    torch.cuda.synchronize()
    from oracle import oracle

    w = min(n, 1 << 20)
    for r0 in sorted({lo, lo + n // 2 - w // 2, hi - w}):
        i0, i1 = merge_coranks(A, B, [r0, r0 + w], torch)
        want = oracle.seq_merge(A[i0:i1].cpu().numpy().view(np.uint64),
                                B[r0 - i0:r0 + w - i1].cpu().numpy().view(np.uint64))
        got = a[r0 - lo:r0 - lo + w].cpu().numpy().view(np.uint64)
        assert np.array_equal(got, want), f"sharded merge parity failed at {r0}"
    assert bool((a[1:] >= a[:-1]).all().item())
    ends = torch.stack([a[0], a[-1]])
    alle = [torch.zeros_like(ends) for _ in range(ws)]
    dist.all_gather(alle, ends)
    assert all(int(alle[r][1]) <= int(alle[r + 1][0]) for r in range(ws - 1)), "shard order"
    del g, A, B
    torch.cuda.empty_cache()
    for _ in range(max(args.warmup - 1, 0)):
        regen()
        step()
    torch.cuda.synchronize()
    barrier(ws)
    clk = ClockSampler(dev)
    ms = regen_timed(step, regen, args.steps, torch, st, ws=ws)
    clocks = clk.stop()
    ms = max_over_ranks(ms, ws)
    per_step = ms / args.steps
    value = n_total * args.steps / (ms / 1e3)
    pk = peaks()
    achieved = 16 * n / (per_step / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": None,
            "note": "per GPU: 16 B/word of its shard algorithmic; the step also rotates shard "
                    "pieces across GPUs (log2(G) levels of P2P mirror swaps)"}
    cfg = {"workload": "in-place merge of two sorted runs, BASELINE configs[3]", "n": n_total,
           "n_per_rank": n, "split": na,
           "values": f"Rng({args.seed}).words >> 34, in [0,2^30), runs sorted (untimed)",
           "l2": "inputs larger than L2; shard restored from a pristine copy between steps "
                 "(untimed)",
           "parallelism": f"shard{ws}: co-ranks + in-place rotations + local merge",
           "check": "oracle windows of each rank's output + global shard order",
           "seed": args.seed}
    return dict(value=value, per_step=per_step, roof=roof, e2e=None, cpu=None, cfg=cfg,
                clocks=clocks, launches=args.steps, extra={})


def run_filter(args, ws, rank, local, torch, pip, lib):
    if ws > 1:
        return run_filter_sharded(args, ws, rank, local, torch, pip, lib)
    n = 1 << (args.log2n or 32)
    dev = local
    st = torch.cuda.current_stream()
    sptr = st.cuda_stream
    a = torch.empty(n, dtype=torch.int64, device=f"cuda:{dev}")
    rng = pip.Rng(args.seed)
    regen = lambda: rng.words_device(0, n, shift=1, device=dev, out=a)  # noqa: E731
    sp, sb = pip.runtime.scratch_for(dev, sptr)
    mdev = torch.zeros(1, dtype=torch.int64, device=f"cuda:{dev}")
    desc = pip.pred.mod_eq(3, 0).descriptor()

    def step():
        rc = lib.pip_filter_u64(a.data_ptr(), n, C.byref(desc), mdev.data_ptr(), sp, sb, sptr)
        assert rc == 0, rc

    # parity of the first (warm-up) step against the oracle on sampled
    # windows (start, middle, end of the input): the kept words of input
    # window [lo, hi) must sit at a[count(src[0:lo)) : ...], in order
    regen()
    src = a.clone()
    step()
    torch.cuda.synchronize()
    pip._lib.check_stall(sp, sptr, "filter")
    m = int(mdev.item())
    check_filter_windows(a, src, m, pip.pred.mod_eq(3, 0), lib, desc, sp, sb, sptr, torch)
    del src
    for _ in range(max(args.warmup - 1, 0)):
        regen()
        step()
    torch.cuda.synchronize()
    clk = ClockSampler(dev)
    ms = regen_timed(step, regen, args.steps, torch, st)
    clocks = clk.stop()
    per_step = ms / args.steps
    value = n * args.steps / (ms / 1e3)
    algo = 8 * n + 8 * m
    pk = peaks()
    achieved = algo / (per_step / 1e3) / 1e9
    tb = ncu_traffic("filter")
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": (tb * n) if tb else None,
            "note": f"8 B/word read + 8 B/kept word written (m/n = {m / n:.4f}); peak = {pk['source']}"}
    e2e = None if args.no_e2e else e2e_host(lib, "filter", n, args, torch, dev, ws)
    cpu = None if args.no_cpu else cpu_baseline("filter", args)
    cfg = {"workload": "stable in-place filter x % 3 == 0, BASELINE configs[2]", "n": n,
           "values": f"Rng({args.seed}).words >> 1, in [0,2^63)", "kept": m,
           "l2": "inputs larger than L2; input regenerated between steps (untimed)",
           "parallelism": "single-GPU", "seed": args.seed}
    # filter_ws2_kernel + the tail kernel when n is not a multiple of the tile
    return dict(value=value, per_step=per_step, roof=roof, e2e=e2e, cpu=cpu, cfg=cfg,
                clocks=clocks, launches=(1 + (1 if n % 6656 else 0)) * args.steps, extra={})


def sort_run(t, torch, pip):
    """Sort a device run of any length (torch.sort stops at INT_MAX elements):
    sort pieces of 2^30 with torch, then merge adjacent pieces in place."""
    n = t.numel()
    piece = 1 << 30
    for s in range(0, n, piece):
        t[s:s + piece] = torch.sort(t[s:s + piece]).values
    width = piece
    while width < n:
        for s in range(0, n, 2 * width):
            e = min(s + 2 * width, n)
            if s + width < e:
                pip.relaxed.merge_relaxed(t[s:e], width)
        width *= 2


def run_partition(args, ws, rank, local, torch, pip, lib):
    if ws > 1:
        raise SystemExit("partition is benchmarked on one GPU")
    n = 1 << (args.log2n or 32)
    dev = local
    st = torch.cuda.current_stream()
    sptr = st.cuda_stream
    a = torch.empty(n, dtype=torch.int64, device=f"cuda:{dev}")
    rng = pip.Rng(args.seed)
    regen = lambda: rng.words_device(0, n, shift=1, device=dev, out=a)  # noqa: E731
    mdev = torch.zeros(1, dtype=torch.int64, device=f"cuda:{dev}")
    p = pip.pred.mod_eq(3, 0)
    desc = p.descriptor()
    wb = lib.pip_partition_workspace_bytes(n)
    wst = torch.empty(max(wb, 16), dtype=torch.uint8, device=f"cuda:{dev}")

    def step():
        rc = lib.pip_partition_u64(a.data_ptr(), n, C.byref(desc), mdev.data_ptr(), wst.data_ptr(),
                                   wb, sptr)
        assert rc == 0, rc

    for _ in range(args.warmup):
        regen()
        step()
    torch.cuda.synchronize()
    m = int(mdev.item())
    # size-independent checks: prefix all true, suffix all false (x % 3 == 0)
    assert bool(((a[:m].view(torch.int64) % 3) == 0).all())
    assert not bool(((a[m:].view(torch.int64) % 3) == 0).any())
    # misfits of this input: false words left of m (= true words right of m)
    regen()
    X = int(((a[:m] % 3) != 0).sum().item())
    clk = ClockSampler(dev)
    ms = regen_timed(step, regen, args.steps, torch, st)
    clocks = clk.stop()
    per_step = ms / args.steps
    value = n * args.steps / (ms / 1e3)
    algo = 8 * n + 16 * X  # every word read once, every misplaced word written once
    pk = peaks()
    achieved = algo / (per_step / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": None,
            "note": f"8 B/word read + 16 B per misfit pair (X/n = {X / n:.4f}); kernels: count, "
                    f"plan, bounds, swap; peak = {pk['source']}"}
    e2e = None if args.no_e2e else e2e_host(lib, "partition", n, args, torch, dev, ws)
    cpu = None if args.no_cpu else cpu_baseline("partition", args)
    cfg = {"workload": "unstable in-place partition x % 3 == 0 (SURVEY 8(f) row 3; configs[2] "
                       "inputs)", "n": n, "values": f"Rng({args.seed}).words >> 1, in [0,2^63)",
           "kept": m, "misfit_pairs": X,
           "l2": "inputs larger than L2; input regenerated between steps (untimed)",
           "parallelism": "single-GPU", "seed": args.seed}
    return dict(value=value, per_step=per_step, roof=roof, e2e=e2e, cpu=cpu, cfg=cfg,
                clocks=clocks, launches=4 * args.steps, extra={})


def run_merge(args, ws, rank, local, torch, pip, lib):
    if ws > 1:
        return run_merge_sharded(args, ws, rank, local, torch, pip, lib)
    n = 1 << (args.log2n or 32)
    na = n // 2
    dev = local
    st = torch.cuda.current_stream()
    sptr = st.cuda_stream
    a = torch.empty(n, dtype=torch.int64, device=f"cuda:{dev}")
    rng = pip.Rng(args.seed)

    def regen():
        rng.words_device(0, n, shift=34, device=dev, out=a)
        sort_run(a[:na], torch, pip)
        sort_run(a[na:], torch, pip)

    budget = pip.EpsilonConfig(0.5)
    b = budget.prefix_words(n)
    wb = lib.pip_merge_workspace_bytes(n, na, b)
    ws_t = torch.empty(max(wb, 16), dtype=torch.uint8, device=f"cuda:{dev}")
    sp, sb = pip.runtime.scratch_for(dev, sptr)

    def step():
        rc = lib.pip_merge_u64(a.data_ptr(), n, na, 0, ws_t.data_ptr(), wb, sp, sb, sptr)
        assert rc == 0, rc

    regen()
    orig = a.clone()
    step()
    torch.cuda.synchronize()
    # parity of the first (warm-up) step: sampled output windows against the
    # oracle's sequential merge of the matching input ranges, plus global
    # sortedness (values < 2^30: signed order = unsigned)
    check_merge_windows(a, orig, na, torch)
    assert bool((a[1:] >= a[:-1]).all().item())
    del orig
    for _ in range(max(args.warmup - 1, 0)):
        regen()
        step()
    clk = ClockSampler(dev)
    ms = regen_timed(step, regen, args.steps, torch, st)
    clocks = clk.stop()
    per_step = ms / args.steps
    value = n * args.steps / (ms / 1e3)
    pk = peaks()
    achieved = 16 * n / (per_step / 1e3) / 1e9
    tb = ncu_traffic("merge")
    two_pass = 32 * n / (per_step / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": (tb * n) if tb else None,
            "two_pass_achieved": round(two_pass, 1),
            "two_pass_frac": round(two_pass / pk["hbm_gbs"], 4),
            "displacement_bound_frac": round(24 * n / (per_step / 1e3) / 1e9 / pk["hbm_gbs"], 4),
            "note": "frac: 16 B/word algorithmic (each word read once, written once).  With "
                    "b(n) = 0.02 n words of workspace and sequential accesses every displaced "
                    "A word must be parked once: >= 24 B/word for equal interleaved runs "
                    "(displacement_bound_frac; DESIGN.md 3.3).  This implementation's two "
                    "parallel passes (chunk permutation + block merge) move 32 B/word; "
                    "two_pass_frac is the kernels' DRAM throughput on those bytes, not a "
                    "lower bound"}
    e2e = None if args.no_e2e else e2e_host(lib, "merge", n, args, torch, dev, ws, budget=b)
    cpu = None if args.no_cpu else cpu_baseline("merge", args)
    cfg = {"workload": "in-place merge of two sorted runs (merge_relaxed, eps=0.5, f=0.02), "
                       "BASELINE configs[3]", "n": n, "split": na,
           "values": f"Rng({args.seed}).words >> 34, in [0,2^30), runs sorted (untimed)",
           "workspace_bytes": wb, "budget_words": b,
           "l2": "inputs larger than L2; runs regenerated + sorted between steps (untimed)",
           "parallelism": "single-GPU", "seed": args.seed}
    return dict(value=value, per_step=per_step, roof=roof, e2e=e2e, cpu=cpu, cfg=cfg,
                clocks=clocks, launches=args.steps, extra={})


def run_rp(args, ws, rank, local, torch, pip, lib, small: bool):
    if ws > 1:
        raise SystemExit("the random permutation is single-GPU (replicas only)")
    dev = local
    st = torch.cuda.current_stream()
    sptr = st.cuda_stream
    if small:
        n = 10 ** 6 if args.log2n is None else 1 << args.log2n
        g = np.random.Generator(np.random.PCG64(args.seed))
        hh = g.integers(0, np.arange(1, n + 1, dtype=np.int64), dtype=np.int64)
        h = torch.from_numpy(hh).cuda()
        hsrc = f"PCG64({args.seed}) integers(0, i+1)"
    else:
        n = 1 << (args.log2n or 30)
        h = torch.empty(n, dtype=torch.int64, device=f"cuda:{dev}")
        pip.Rng(args.seed).swaps_device(0, n, device=dev, out=h)
        hsrc = f"make_swap_sequence(n, Rng({args.seed})) generated on device"
    a = torch.arange(n, dtype=torch.int64, device=f"cuda:{dev}")
    budget = pip.EpsilonConfig(0.5)
    prefix = budget.prefix_words(n)
    wb = lib.pip_rp_workspace_bytes(n, prefix, 3)
    ws_t = torch.empty(wb, dtype=torch.uint8, device=f"cuda:{dev}")
    stats = pip._lib.PipRpStats()
    counts = np.zeros(1 << 16, dtype=np.uint64)

    def step():
        rc = lib.pip_random_permutation_u64(a.data_ptr(), h.data_ptr(), n, prefix, 3, 0,
                                            counts.ctypes.data, len(counts), None,
                                            ws_t.data_ptr(), wb, C.byref(stats), sptr)
        assert rc == 0, rc

    step()
    torch.cuda.synchronize()
    # parity of the first step, every word, at every size (C4 included):
    # the oracle's sequential Knuth shuffle (baselines.py:44-54) in C
    from oracle import oracle

    ref = np.arange(n, dtype=np.uint64)
    oracle.seq_knuth_shuffle(ref, h.cpu().numpy().view(np.uint64))
    assert np.array_equal(a.cpu().numpy().view(np.uint64), ref), "permutation parity failed"
    a.copy_(torch.arange(n, dtype=torch.int64, device=f"cuda:{dev}"))
    for _ in range(max(args.warmup - 1, 0)):
        step()
    torch.cuda.synchronize()
    clk = ClockSampler(dev)
    ms = Events(torch).time(step, args.steps, st)
    clocks = clk.stop()
    per_step = ms / args.steps
    value = n * args.steps / (ms / 1e3)
    iters = int(stats.n_iterates)
    # roofline: one random 8-byte read-modify-write (a 32-byte sector) per
    # committed swap, against a measured random-RMW rate on an equal array
    bufn = n
    buf = torch.zeros(bufn, dtype=torch.int64, device=f"cuda:{dev}")
    msf = C.c_float(0)
    upd = max(bufn, 1 << 26)
    # both request forms: load + store, and one atomic exchange per update
    # (the faster of the two is the ceiling the swaps are held against)
    rates = []
    for form in (0, 1):
        assert lib.pip_bench_random_update(buf.data_ptr(), bufn, upd, 7, form, C.byref(msf), sptr) == 0
        rates.append(upd / (msf.value / 1e3))
    rmw_rate = max(rates)
    del buf
    swaps_rate = iters / (per_step / 1e3)
    tb = None if small else ncu_traffic("rp")
    roof = {"bound": "hbm", "achieved": round(swaps_rate * 32 / 1e9, 1),
            "peak": round(rmw_rate * 32 / 1e9, 1), "unit": "GB/s",
            "frac": round(swaps_rate / rmw_rate, 4), "traffic": (tb * n) if tb else None,
            "frac_vs_load_store": round(swaps_rate / rates[0], 4),
            "note": "random-sector roofline: one 32-B sector RMW per committed swap "
                    f"({iters} swaps) vs measured random 8-B updates over {bufn} words: "
                    f"atomic exchange {rates[1] / 1e9:.2f} G/s (the peak), load + store "
                    f"{rates[0] / 1e9:.2f} G/s (round 1's denominator)"}
    e2e = None
    if not args.no_e2e:
        e2e = e2e_host(lib, "rp", n, args, torch, dev, ws, h=h, prefix=prefix, ref=ref)
    del ref
    cpu = None if args.no_cpu else cpu_baseline("rp0" if small else "rp", args)
    cfg = {"workload": ("random permutation n=10^6, BASELINE configs[0]" if small else
                        "random permutation n=2^30, BASELINE configs[4]"),
           "n": n, "H": hsrc, "variant": "final", "budget": "EpsilonConfig(0.5, 0.02)",
           "prefix": prefix, "rounds": int(stats.rounds), "workspace_bytes": wb,
           "workspace_words_over_b": round(wb / 8 / prefix, 3),
           "l2": "C0 is L2-resident by design (8 MB); C4 arrays 8 GiB >> L2",
           "parallelism": "single-GPU", "seed": args.seed}
    # the validation pass (non-self counts) + the persistent round kernel
    return dict(value=value, per_step=per_step, roof=roof, e2e=e2e, cpu=cpu, cfg=cfg,
                clocks=clocks, launches=2 * args.steps, extra={})


# ---------------------------------------------------------------------------
# end to end through the C ABI with host buffers (pinned), copies timed

def e2e_host(lib, op, n, args, torch, dev, ws, **kw):
    steps = max(2, min(args.steps, 3))
    try:
        host = torch.empty(n, dtype=torch.int64, pin_memory=True)
    except RuntimeError as exc:
        return {"value": None, "unit": "elements/s", "error": f"pinned alloc failed: {exc}"}
    hp = host.data_ptr()
    rng_seed = args.seed
    d = torch.empty(n, dtype=torch.int64, device=f"cuda:{dev}")

    def fill():
        import paper_2103_01216_b200 as pip

        if op == "scan":
            pip.Rng(rng_seed).words_device(0, n, shift=44, device=dev, out=d)
        elif op in ("filter", "partition"):
            pip.Rng(rng_seed).words_device(0, n, shift=1, device=dev, out=d)
        elif op == "merge":
            pip.Rng(rng_seed).words_device(0, n, shift=34, device=dev, out=d)
            sort_run(d[: n // 2], torch, pip)
            sort_run(d[n // 2:], torch, pip)
        else:
            d.copy_(torch.arange(n, dtype=torch.int64, device=f"cuda:{dev}"))
        host.copy_(d)
        torch.cuda.synchronize()

    hh = None
    if op == "rp":
        hh = torch.empty(n, dtype=torch.int64, pin_memory=True)
        hh.copy_(kw["h"])
    total = 0.0
    bi = bo = 0
    out = C.c_uint64(0)
    for it in range(steps + 1):  # the first call is an untimed warm-up (pools, pinned staging)
        fill()
        t0 = time.perf_counter()
        if op == "scan":
            out = C.c_uint64(0)
            rc = lib.pip_scan_u64_host(hp, n, 0, 0, 1, C.byref(out), dev)
            bi, bo = 8 * n, 8 * n
        elif op == "filter":
            import paper_2103_01216_b200 as pip

            desc = pip.pred.mod_eq(3, 0).descriptor()
            out = C.c_uint64(0)
            rc = lib.pip_filter_u64_host(hp, n, C.byref(desc), C.byref(out), dev)
            bi, bo = 8 * n, 8 * int(out.value)
        elif op == "merge":
            rc = lib.pip_merge_u64_host(hp, n, n // 2, kw["budget"], dev)
            bi, bo = 8 * n, 8 * n
        elif op == "partition":
            import paper_2103_01216_b200 as pip

            desc = pip.pred.mod_eq(3, 0).descriptor()
            out = C.c_uint64(0)
            rc = lib.pip_partition_u64_host(hp, n, C.byref(desc), C.byref(out), dev)
            bi, bo = 8 * n, 8 * n
        else:
            import paper_2103_01216_b200 as pip

            stats = pip._lib.PipRpStats()
            rc = lib.pip_random_permutation_u64_host(hp, hh.data_ptr(), n, kw["prefix"], 3,
                                                     C.byref(stats), dev)
            bi, bo = 16 * n, 8 * n
        if it > 0:
            total += time.perf_counter() - t0
        assert rc == 0, rc
    # parity of the last timed call's output (d still holds its input)
    check_e2e(op, host, d, out.value if op in ("scan", "filter", "partition") else None, n,
              torch, kw)
    del d
    return {"value": n * steps / total, "unit": "elements/s", "h2d_bytes_per_step": bi,
            "d2h_bytes_per_step": bo, "steps": steps, "checked": True,
            "note": "synchronous C-ABI *_host call on pinned host memory; wall clock "
                    "around the call (H2D + kernels + D2H); the last call's output is "
                    "checked against the oracle on sampled windows (the permutation: "
                    "every word)"}


def check_e2e(op, host, d, result, n, torch, kw):
    import paper_2103_01216_b200 as pip
    from oracle import oracle

    if op == "scan":
        src = d
        for lo, hi in _windows(n):
            carry = 0 if lo == 0 else int(host[lo - 1].item()) & ((1 << 64) - 1)
            want, _ = oracle.seq_scan(src[lo:hi].cpu().numpy().view(np.uint64), init=carry,
                                      inclusive=True)
            got = host[lo:hi].numpy().view(np.uint64)
            assert np.array_equal(got, want), f"e2e scan parity failed on window [{lo}, {hi})"
        assert int(host[n - 1].item()) & ((1 << 64) - 1) == result, "e2e scan total"
    elif op in ("filter", "partition"):
        dev = d.device.index
        st = torch.cuda.current_stream().cuda_stream
        sp, sb = pip.runtime.scratch_for(dev, st)
        lib = pip._lib.load()
        p = pip.pred.mod_eq(3, 0)
        desc = p.descriptor()
        if op == "filter":
            check_filter_windows(host, d, result, p, lib, desc, sp, sb, st, torch)
        else:
            cnt = torch.zeros(1, dtype=torch.int64, device=d.device)
            assert lib.pip_count_u64(d.data_ptr(), n, C.byref(desc), cnt.data_ptr(), sp, sb, st) == 0
            m = int(cnt.item())
            assert m == result, "e2e partition count"
            for lo, hi in _windows(n):
                x = host[lo:hi].numpy().view(np.uint64)
                keep = (x % np.uint64(3)) == 0
                assert bool(np.all(keep[: max(0, m - lo)])) and not bool(np.any(keep[max(0, m - lo):])), \
                    f"e2e partition contract failed on window [{lo}, {hi})"
    elif op == "merge":
        check_merge_windows(host, d, n // 2, torch)
    else:
        assert np.array_equal(host.numpy().view(np.uint64), kw["ref"]), "e2e permutation parity"



# ---------------------------------------------------------------------------
# CPU baseline: the C port of the reference's own algorithm (oracle/)

CPU_SAMPLE_LOG2 = {"scan": 28, "filter": 28, "merge": 26, "rp": 24, "rp0": None, "partition": 26}


def _cpu_input(op, n, seed):
    import paper_2103_01216_b200 as pip

    rng = pip.Rng(seed)
    if op == "scan":
        return rng.words(0, n) >> np.uint64(44), None
    if op in ("filter", "partition"):
        return rng.words(0, n) >> np.uint64(1), None
    if op == "merge":
        x = rng.words(0, n) >> np.uint64(34)
        x[: n // 2].sort()
        x[n // 2:].sort()
        return x, None
    if op == "rp0":
        g = np.random.Generator(np.random.PCG64(seed))
        h = g.integers(0, np.arange(1, n + 1, dtype=np.int64), dtype=np.int64).astype(np.uint64)
        return np.arange(n, dtype=np.uint64), h
    h = rng.words(0, n) % (np.arange(n, dtype=np.uint64) + np.uint64(1))
    return np.arange(n, dtype=np.uint64), h


def cpu_run(op, x, h, threads):
    import paper_2103_01216_b200 as pip
    from oracle import oracle

    n = len(x)
    if op == "scan":
        oracle.ref_scan(x, threads)
    elif op == "filter":
        oracle.ref_filter_kway(x, pip.pred.mod_eq(3, 0), threads)
    elif op == "merge":
        oracle.ref_merge_strong(x, n // 2, threads)
    elif op == "partition":
        oracle.ref_partition_unstable(x, pip.pred.mod_eq(3, 0))  # sequential, as the reference
    else:
        oracle.ref_random_permutation(x, h, pip.EpsilonConfig(0.5).prefix_words(n), "final",
                                      threads)


def cpu_baseline(op, args, budget_s: float = 10.0) -> dict:
    from oracle import oracle

    oracle.build()
    lg = CPU_SAMPLE_LOG2[op]
    n = 10 ** 6 if lg is None else 1 << lg
    threads = cpu_threads()
    x0, h = _cpu_input(op, n, args.seed)
    reps, el = 0, 0.0
    while el < budget_s and reps < 2000:  # about 10 s of CPU work (time-bounded sample)
        x = x0.copy()
        t0 = time.perf_counter()
        cpu_run(op, x, h, threads)
        el += time.perf_counter() - t0
        reps += 1
    names = {"scan": "strong.scan (Alg. 3 up/down sweep)", "filter": "strong.filter_kway",
             "merge": "strong.merge_strong", "rp": "relaxed.random_permutation (final)",
             "rp0": "relaxed.random_permutation (final)",
             "partition": "strong.partition_unstable (sequential, as the reference)"}
    if op == "partition":
        threads = 1
    return {"value": n * reps / el, "unit": "elements/s", "cores": threads, "kind": "port",
            "sample": f"{names[op]} C/OpenMP port (oracle/pip_oracle.c) on n={n} "
                      f"words x {reps} reps, {el:.1f} s, same generator/seed"}


# ---------------------------------------------------------------------------

def main():
    args = parse()
    ws, rank, local = dist_init()
    metric = "elements/s per in-place op (perm/scan/filter/merge); % of HBM roofline"
    if args.impl == "reference":
        if rank != 0:
            barrier(ws) if False else None
            return
        op = args.op
        lg = CPU_SAMPLE_LOG2[op]
        n = 10 ** 6 if lg is None else 1 << lg
        threads = cpu_threads()
        x0, h = _cpu_input(op, n, args.seed)
        for _ in range(args.warmup):
            cpu_run(op, x0.copy(), h, threads)
        el = 0.0
        for _ in range(args.steps):
            x = x0.copy()
            t0 = time.perf_counter()
            cpu_run(op, x, h, threads)
            el += time.perf_counter() - t0
        value = n * args.steps / el
        full = {"scan": 1 << 32, "filter": 1 << 32, "merge": 1 << 32, "rp": 1 << 30, "rp0": 10 ** 6,
                "partition": 1 << 32}
        line = {"metric": metric, "value": value, "unit": "elements/s", "impl": "reference",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
                "scaling": "strong" if op in ("scan", "filter", "merge") else "weak",
                "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": {"workload": {"scan": "inclusive in-place scan, BASELINE configs[1]",
                                        "filter": "stable filter x%3==0, BASELINE configs[2]",
                                        "merge": "in-place merge, BASELINE configs[3]",
                                        "rp": "random permutation, BASELINE configs[4]",
                                        "rp0": "random permutation, BASELINE configs[0]",
                                        "partition": "unstable in-place partition x%3==0 "
                                                     "(SURVEY 8(f) row 3)"}[op],
                           "n": full[op], "sample_n": n, "seed": args.seed},
                "cpu_baseline": {"value": value, "unit": "elements/s", "cores": threads,
                                 "kind": "port",
                                 "sample": f"C/OpenMP port of the reference algorithm "
                                           f"(oracle/pip_oracle.c), n={n} per step"},
                "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    import paper_2103_01216_b200 as pip

    torch.cuda.set_device(local)
    lib = pip._lib.load()
    if args.op == "scan":
        r = run_scan(args, ws, rank, local, torch, pip, lib)
    elif args.op == "filter":
        r = run_filter(args, ws, rank, local, torch, pip, lib)
    elif args.op == "merge":
        r = run_merge(args, ws, rank, local, torch, pip, lib)
    elif args.op == "partition":
        r = run_partition(args, ws, rank, local, torch, pip, lib)
    else:
        r = run_rp(args, ws, rank, local, torch, pip, lib, small=(args.op == "rp0"))
    if rank == 0:
        e2e = r["e2e"]
        line = {"metric": metric, "value": r["value"], "unit": "elements/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["per_step"],
                "higher_is_better": True,
                "scaling": "strong" if args.op in ("scan", "filter", "merge") else "weak",
                "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": r["cfg"], "roofline": r["roof"], "cpu_baseline": r["cpu"],
                "e2e": e2e, "clocks": r["clocks"], "gpu_launches": r["launches"],
                "paper_72core_elements_per_s": PAPER_GELEM_S.get(args.op)}
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
