"""Sharded scan / filter / merge over ``torch.distributed`` (one process per GPU).

The reference has no distributed code; this is the
multi-GPU extension the BASELINE north star asks for.  An
array of n words is sharded evenly: rank r owns global words
[r*S, (r+1)*S), S = n / world (the last rank may own fewer).

  sharded_scan    local fold -> all_gather of shard totals (8 B per rank) ->
                  exclusive carry -> in-place scan with a DEVICE carry-in.
                  Fully in place; 24 B/word of HBM traffic (fold + scan).
  sharded_filter  local stable compaction -> all_gather of kept counts ->
                  every rank's kept words move to global [O_r, O_r + c_r)
                  (destinations precede sources: the reference's batching
                  rule, strong.py:317-327, at rank granularity) through one
                  all_to_all; ranks beyond the packed prefix keep an
                  unspecified tail, as in the reference.
  sharded_merge   global merge-path co-ranks at the shard boundaries by a
                  batched collective binary search (log2(n) tiny all_reduces) ->
                  one all_to_all that brings every rank its A and B pieces ->
                  local in-place merge.
The local kernels are pluggable (``LocalOps``): ``CudaOps`` runs libpip on
the rank's GPU (NCCL moves device buffers); tests drive the same plan on CPU
tensors with gloo and a numpy stand-in for the local ops.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

M64 = (1 << 64) - 1

__all__ = ["LocalOps", "CudaOps", "shard_bounds", "sharded_scan", "sharded_filter",
           "sharded_merge"]


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    s = (n + world - 1) // world
    lo = min(rank * s, n)
    return lo, min(lo + s, n)


class LocalOps:
    """Local (per-rank) in-place kernels the sharded algorithms are built on."""

    device: torch.device

    def reduce(self, t: torch.Tensor) -> torch.Tensor:  # [1] int64 (u64 bits)
        raise NotImplementedError

    def scan_carry(self, t: torch.Tensor, carry: torch.Tensor, inclusive: bool) -> None:
        raise NotImplementedError

    def filter(self, t: torch.Tensor, pred) -> int:
        raise NotImplementedError

    def merge(self, t: torch.Tensor, split: int) -> None:
        raise NotImplementedError


class CudaOps(LocalOps):
    """libpip on the current CUDA device/stream (the product path)."""

    def __init__(self):
        from . import _lib

        self.lib = _lib.load()
        self.device = torch.device("cuda", torch.cuda.current_device())

    def _st(self):
        from .runtime import scratch_for

        st = torch.cuda.current_stream().cuda_stream
        return st, scratch_for(self.device.index, st)

    def reduce(self, t):
        from . import _lib

        st, (sp, sb) = self._st()
        out = torch.zeros(1, dtype=torch.int64, device=self.device)
        _lib.check(self.lib.pip_reduce_u64(t.data_ptr(), t.numel(), 0, out.data_ptr(), sp, sb, st),
                   "reduce")
        _lib.check_stall(sp, st, "reduce")
        return out

    def scan_carry(self, t, carry, inclusive):
        from . import _lib

        st, (sp, sb) = self._st()
        tot = torch.zeros(1, dtype=torch.int64, device=self.device)
        _lib.check(self.lib.pip_scan_u64_carry(t.data_ptr(), t.numel(), 0, 0, int(inclusive),
                                               carry.data_ptr(), tot.data_ptr(), sp, sb, st),
                   "scan")
        _lib.check_stall(sp, st, "scan")

    def filter(self, t, pred):
        from . import strong

        return strong.filter_kway(t, pred)

    def merge(self, t, split):
        from . import relaxed

        relaxed.merge_relaxed(t, split)


def _u64sum(x: torch.Tensor) -> int:
    return int(np.asarray(x.cpu().numpy(), dtype=np.int64).view(np.uint64).sum(dtype=np.uint64))


def sharded_scan(local: torch.Tensor, ops: LocalOps, inclusive: bool = True, group=None) -> int:
    """In-place prefix sum (mod 2^64) of the global array; returns the total."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    tot = ops.reduce(local)
    gathered = [torch.zeros_like(tot) for _ in range(world)]
    dist.all_gather(gathered, tot, group=group)
    allt = torch.cat(gathered)
    carry = allt[:rank].sum(dim=0, keepdim=True) if rank else torch.zeros_like(tot)
    ops.scan_carry(local, carry, inclusive)
    return _u64sum(allt) & M64


def sharded_filter(local: torch.Tensor, n_global: int, pred, ops: LocalOps, group=None) -> int:
    """Stable filter of the global array: global a[0:m) = kept words in order.

    Returns m.  Words beyond the packed prefix are unspecified.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    c = ops.filter(local, pred)  # local stable compaction: local[0:c)
    cnt = torch.tensor([c], dtype=torch.int64, device=local.device)
    gathered = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(gathered, cnt, group=group)
    counts = [int(g.item()) for g in gathered]
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    m = int(offs[-1])
    bounds = [shard_bounds(n_global, world, r) for r in range(world)]
    # send plan: my kept words [offs[r], offs[r] + c) split by destination shard
    send = []
    for d in range(world):
        lo, hi = bounds[d]
        a0, a1 = max(lo, int(offs[rank])), min(hi, int(offs[rank]) + c)
        send.append(max(0, a1 - a0))
    recv = []
    mylo, myhi = bounds[rank]
    for s in range(world):
        a0, a1 = max(mylo, int(offs[s])), min(myhi, int(offs[s]) + counts[s])
        recv.append(max(0, a1 - a0))
    src = local[:c].clone() if c else local[:0].clone()
    out = torch.empty(sum(recv), dtype=local.dtype, device=local.device)
    _all_to_all(out, src, recv, send, group)
    if sum(recv):
        # the packed prefix covers global [0, m): my share is [mylo, min(myhi, m)),
        # received in source-rank order, i.e. in global order
        local[:sum(recv)] = out
    return m


def _all_to_all(out, inp, recv_splits, send_splits, group):
    """all_to_all_single with split lists (gloo has it; falls back to p2p)."""
    try:
        dist.all_to_all_single(out, inp, output_split_sizes=recv_splits,
                               input_split_sizes=send_splits, group=group)
        return
    except (RuntimeError, NotImplementedError):
        pass
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    so = np.concatenate([[0], np.cumsum(send_splits)]).astype(np.int64)
    ro = np.concatenate([[0], np.cumsum(recv_splits)]).astype(np.int64)
    reqs = []
    for peer in range(world):
        if peer == rank:
            if send_splits[peer]:
                out[ro[peer]:ro[peer + 1]] = inp[so[peer]:so[peer + 1]]
            continue
        if send_splits[peer]:
            reqs.append(dist.isend(inp[so[peer]:so[peer + 1]].contiguous(), peer, group=group))
        if recv_splits[peer]:
            buf = torch.empty(int(recv_splits[peer]), dtype=out.dtype, device=out.device)
            reqs.append((dist.irecv(buf, peer, group=group), buf, peer))
    for r in reqs:
        if isinstance(r, tuple):
            r[0].wait()
            out[ro[r[2]]:ro[r[2] + 1]] = r[1]
        else:
            r.wait()


def _coranks(local, lo, n, na, qs, group) -> list[int]:
    """Merge-path co-ranks at output positions qs over A = g[0:na), B = g[na:n)
    (A first on ties): a batched binary search, one all_reduce per step in
    which the owner of each probed word contributes it."""
    nb = n - na
    ilo = np.array([max(0, q - nb) for q in qs], dtype=np.int64)
    ihi = np.array([min(q, na) for q in qs], dtype=np.int64)
    qv = np.array(qs, dtype=np.int64)
    hi_excl = lo + local.numel()
    host = local.cpu().numpy() if local.device.type == "cpu" else None
    while np.any(ilo < ihi):
        mid = (ilo + ihi) // 2
        probe = np.concatenate([mid, na + (qv - mid - 1)])
        active = np.concatenate([ilo < ihi, ilo < ihi])
        vals = torch.zeros(len(probe), dtype=torch.int64, device=local.device)
        mine = active & (probe >= lo) & (probe < hi_excl)
        if mine.any():
            idx = torch.from_numpy(probe[mine] - lo).to(local.device)
            vals[torch.from_numpy(np.flatnonzero(mine)).to(local.device)] = (
                local[idx] if host is None else torch.from_numpy(host[probe[mine] - lo]))
        dist.all_reduce(vals, op=dist.ReduceOp.SUM, group=group)
        v = vals.cpu().numpy().view(np.uint64)
        k = len(qs)
        act = ilo < ihi
        take = (v[:k] <= v[k:]) & act
        ilo, ihi = np.where(take, mid + 1, ilo), np.where(act & ~take, mid, ihi)
    return [int(x) for x in ilo]


def sharded_merge(local: torch.Tensor, n_global: int, split: int, ops: LocalOps,
                  group=None) -> None:
    """Merge the sorted runs g[0:split) and g[split:n) of the sharded array."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bounds = [shard_bounds(n_global, world, r) for r in range(world)]
    lo, hi = bounds[rank]
    # every rank's output boundary co-ranks (computed collectively, all ranks
    # walk the same sequence of probes)
    cr = _coranks(local, lo, n_global, split, [b[0] for b in bounds] + [n_global], group)
    # my output [lo, hi) = A[cr[rank]:cr[rank+1]) + B[lo - cr[rank] : hi - cr[rank+1])
    # send plan: for every destination d, the A and B words I own that d needs
    send, pieces = [], []
    for d in range(world):
        dlo, dhi = bounds[d]
        ia0, ia1 = cr[d], cr[d + 1]                         # A indices for d
        ib0, ib1 = split + dlo - cr[d], split + dhi - cr[d + 1]  # global B positions
        cnt = 0
        for g0, g1 in ((ia0, ia1), (ib0, ib1)):
            a0, a1 = max(g0, lo), min(g1, hi)
            if a1 > a0:
                pieces.append(local[a0 - lo:a1 - lo])
                cnt += a1 - a0
        send.append(cnt)
    recv = []
    for s in range(world):
        slo, shi = bounds[s]
        cnt = 0
        for g0, g1 in ((cr[rank], cr[rank + 1]),
                       (split + lo - cr[rank], split + hi - cr[rank + 1])):
            a0, a1 = max(g0, slo), min(g1, shi)
            cnt += max(0, a1 - a0)
        recv.append(cnt)
    src = torch.cat(pieces) if pieces else local[:0].clone()
    out = torch.empty(hi - lo, dtype=local.dtype, device=local.device)
    _all_to_all(out, src, recv, send, group)
    # received in source-rank order; A words (lower global positions) of each
    # source precede its B words, and sources ascend: rebuild [A piece | B piece]
    na_mine = cr[rank + 1] - cr[rank]
    a_parts, b_parts = [], []
    pos = 0
    for s in range(world):
        slo, shi = bounds[s]
        ga = max(0, min(cr[rank + 1], shi) - max(cr[rank], slo))
        gb = max(0, min(split + hi - cr[rank + 1], shi) - max(split + lo - cr[rank], slo))
        if ga:
            a_parts.append(out[pos:pos + ga])
        pos += ga
        if gb:
            b_parts.append(out[pos:pos + gb])
        pos += gb
    merged_in = torch.cat(a_parts + b_parts) if (a_parts or b_parts) else out[:0]
    local[:] = merged_in
    ops.merge(local, na_mine)
