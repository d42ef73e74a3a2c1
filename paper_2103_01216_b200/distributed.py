"""Sharded scan / filter / merge over ``torch.distributed`` (one process per GPU).

The reference has no distributed code; this is the
multi-GPU extension the BASELINE north star asks for.  An
array of n words is sharded evenly: rank r owns global words
[r*S, (r+1)*S), S = ceil(n / world) (the last rank may own fewer).  All
three are IN PLACE: no rank ever holds a copy of its shard; the only
auxiliary memory is a bounded exchange ring (``wave_words``) and O(world)
descriptors.

  sharded_scan    local fold -> all_gather of shard totals (8 B per rank) ->
                  exclusive carry -> in-place scan with a DEVICE carry-in.
                  24 B/word of HBM traffic (fold + scan), no data exchange.
  sharded_filter  local stable in-place filter -> all_gather of kept counts
                  -> every rank's kept words move to global [O_r, O_r + c_r),
                  which lies at or below its own shard (destination precedes
                  source: strong.py:317-327's batching rule at rank
                  granularity).  Rank r first sends the head of its kept
                  words that belongs to lower shards straight out of its
                  array (no staging), then shifts the rest down in place
                  (pip_move_u64, one pass), and only then receives the
                  words of higher ranks straight into their final slots —
                  which lie above what it kept.  Every wait points to a
                  lower rank, so the chain resolves from rank 0 upwards.
  sharded_merge   merge-path co-ranks of every shard boundary (strong.py:
                  474-488) by a 4096-ary collective search: one all_reduce
                  of sampled probe words per level, 3 levels for 2^32 words
                  (instead of ~32 bisection steps) -> the block interleave
                  A_0..A_{G-1} B_0..B_{G-1} -> A_0 B_0 .. A_{G-1} B_{G-1}
                  (A_d, B_d = the run pieces output shard d needs) by
                  recursive rotations (the reference's merge_strong step,
                  strong.py:496-522, at shard granularity), each rotation
                  three reversals, each reversal pairwise mirror swaps in
                  waves through a bounded ring -> local in-place merge of
                  [A_d | B_d].
The local kernels are pluggable (``LocalOps``): ``CudaOps`` runs libpip on
the rank's GPU (NCCL or gloo moves device buffers); the CPU tests drive the
same plans with gloo and a torch stand-in for the local ops.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

M64 = (1 << 64) - 1
SEARCH_FANOUT = 4096
WAVE_WORDS = 1 << 22  # exchange ring per rank (32 MiB)

__all__ = ["LocalOps", "CudaOps", "shard_bounds", "sharded_scan", "sharded_filter",
           "sharded_merge", "merge_coranks"]


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

    def move(self, t: torch.Tensor, dst: int, src: int, length: int) -> None:
        """memmove inside t: t[dst:dst+length] = old t[src:src+length]."""
        raise NotImplementedError

    def reverse(self, t: torch.Tensor) -> None:
        """Reverse t in place."""
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

    def move(self, t, dst, src, length):
        from . import _lib

        if length <= 0 or dst == src:
            return
        st, (sp, sb) = self._st()
        _lib.check(self.lib.pip_move_u64(t.data_ptr(), dst, src, length, sp, sb, st), "move")
        _lib.check_stall(sp, st, "move")

    def reverse(self, t):
        from . import _lib

        if t.numel() > 1:
            st = torch.cuda.current_stream().cuda_stream
            _lib.check(self.lib.pip_reverse_u64(t.data_ptr(), t.numel(), st), "reverse")


def _u64sum(x: torch.Tensor) -> int:
    return int(np.asarray(x.cpu().numpy(), dtype=np.int64).view(np.uint64).sum(dtype=np.uint64))


def _sync(t: torch.Tensor) -> None:
    if t.is_cuda:
        torch.cuda.current_stream(t.device).synchronize()


def _exchange(sends, recvs, group) -> None:
    """Post all sends and receives of one step together and wait.  sends /
    recvs: lists of (peer, tensor view); views are contiguous slices of the
    callers' arrays, so nothing is staged."""
    sends = [(p, t) for p, t in sends if t.numel()]
    recvs = [(p, t) for p, t in recvs if t.numel()]
    if not sends and not recvs:
        return
    staged = []
    if dist.get_backend(group) == "gloo" and any(t.is_cuda for _, t in sends + recvs):
        # gloo moves host buffers only: stage device views through the host
        sends = [(p, t.cpu()) for p, t in sends]
        staged = [(t, torch.empty(t.numel(), dtype=t.dtype)) for _, t in recvs]
        recvs = [(p, h) for (p, _), (_, h) in zip(recvs, staged)]
    ops = [dist.P2POp(dist.isend, t, peer, group) for peer, t in sends]
    ops += [dist.P2POp(dist.irecv, t, peer, group) for peer, t in recvs]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    for dev, h in staged:
        dev.copy_(h)


# ---------------------------------------------------------------------------
# scan

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


# ---------------------------------------------------------------------------
# filter

def filter_plan(counts: list[int], n: int, world: int, rank: int):
    """Movement plan of the sharded filter for ``rank``.

    Returns (down, stay, up): ``down`` = [(dest rank, local lo, local hi,
    dest local lo)] pieces of my kept words local[0:x) that go to lower
    shards; ``stay`` = (src lo, length) of the kept words that stay (moved to
    local 0); ``up`` = [(src rank, dest local lo, length)] pieces higher
    ranks send me, ascending.
    """
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    bounds = [shard_bounds(n, world, r) for r in range(world)]
    lo, hi = bounds[rank]
    o, c = int(offs[rank]), counts[rank]
    x = min(c, max(0, lo - o))  # my kept words landing below my shard
    down = []
    for e in range(rank):
        elo, ehi = bounds[e]
        g0, g1 = max(o, elo), min(o + x, ehi)
        if g1 > g0:
            down.append((e, g0 - o, g1 - o, g0 - elo))
    stay = (x, c - x)
    up = []
    for s in range(rank + 1, world):
        g0, g1 = max(int(offs[s]), lo), min(int(offs[s]) + counts[s], hi)
        if g1 > g0:
            up.append((s, g0 - lo, g1 - g0))
    return down, stay, up


def sharded_filter(local: torch.Tensor, n_global: int, pred, ops: LocalOps, group=None) -> int:
    """Stable filter of the global array, in place: global a[0:m) = the kept
    words in order.  Returns m; words beyond the packed prefix are
    unspecified (as in the reference)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    c = ops.filter(local, pred)  # local stable compaction: local[0:c)
    cnt = torch.tensor([c], dtype=torch.int64, device=local.device)
    gathered = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(gathered, cnt, group=group)
    counts = [int(g.item()) for g in gathered]
    down, (s0, slen), up = filter_plan(counts, n_global, world, rank)
    # 1. the head of my kept words goes to lower shards, straight from my array
    _exchange([(e, local[a:b]) for e, a, b, _ in down], [], group)
    # 2. what stays moves down to local 0 (one in-place pass)
    if slen and s0:
        ops.move(local, 0, s0, slen)
    _sync(local)
    # 3. higher ranks' words land above what I kept, in their final slots
    _exchange([], [(s, local[d:d + ln]) for s, d, ln in up], group)
    _sync(local)
    return sum(counts)


# ---------------------------------------------------------------------------
# merge: co-ranks

def _fetch(local: torch.Tensor, lo: int, positions: np.ndarray, group) -> np.ndarray:
    """Words at the given global positions (-1 = none): one all_reduce in
    which each position's owner contributes its word."""
    vals = torch.zeros(len(positions), dtype=torch.int64, device=local.device)
    mine = (positions >= lo) & (positions < lo + local.numel())
    if mine.any():
        idx = torch.from_numpy(positions[mine] - lo).to(local.device)
        sel = torch.from_numpy(np.flatnonzero(mine)).to(local.device)
        vals[sel] = local[idx]
    dist.all_reduce(vals, op=dist.ReduceOp.SUM, group=group)
    return vals.cpu().numpy().view(np.uint64)


def merge_coranks(local: torch.Tensor, lo: int, n: int, na: int, qs: list[int], group,
                  fanout: int = SEARCH_FANOUT) -> list[int]:
    """Merge-path co-ranks i(q) over A = g[0:na), B = g[na:n) at output
    positions qs (ties from A: the smallest i with i + j = q such that not
    (j > 0 and i < na and B[j-1] >= A[i]), strong.py:474-488).

    Every query's bracket [ilo, ihi] shrinks by ``fanout`` per level: the
    predicate "B[q-i-1] >= A[i]" (monotone in i) is evaluated at up to
    ``fanout`` points of every bracket with ONE all_reduce that fetches all
    probed words; ceil(log_fanout(n)) levels in all.
    """
    nb = n - na
    q = np.array(qs, dtype=np.int64)
    ilo = np.maximum(0, q - nb)   # invariant: P(i) true for i < ilo, false at ihi
    ihi = np.minimum(q, na)
    while np.any(ilo < ihi):
        pts = []
        for k in range(len(q)):
            if ilo[k] < ihi[k]:
                width = ihi[k] - ilo[k]
                step = max(1, -(-width // fanout))
                p = np.arange(ilo[k], ihi[k], step, dtype=np.int64)
            else:
                p = np.empty(0, dtype=np.int64)
            pts.append(p)
        sizes = [len(p) for p in pts]
        allp = np.concatenate(pts) if pts else np.empty(0, dtype=np.int64)
        qk = np.repeat(q, sizes)
        pos = np.concatenate([allp, na + (qk - allp - 1)])
        v = _fetch(local, lo, pos, group)
        m = len(allp)
        true = v[m:] >= v[:m]  # B[q-i-1] >= A[i]  -> the co-rank lies right of i
        at = 0
        for k in range(len(q)):
            if sizes[k]:
                t = true[at:at + sizes[k]]
                p = pts[k]
                # first false probe bounds from above; the last true one + 1 from below
                f = np.flatnonzero(~t)
                nhi = int(p[f[0]]) if len(f) else int(ihi[k])
                tt = np.flatnonzero(t[: f[0]] if len(f) else t)
                nlo = int(p[tt[-1]]) + 1 if len(tt) else int(ilo[k])
                ilo[k], ihi[k] = nlo, nhi
            at += sizes[k]
    return [int(x) for x in ilo]


# ---------------------------------------------------------------------------
# merge: distributed reversal / rotation

def _reverse_range(local: torch.Tensor, lo: int, S: int, x: int, z: int, ops: LocalOps, group,
                   ring: torch.Tensor) -> None:
    """Reverse the global range [x, z) in place: position p <-> x + z - 1 - p
    (shards of S words; rank e owns [e*S, (e+1)*S)).  Pairs that straddle two
    ranks are swapped in waves through ``ring``: this rank's chunk is sent
    while the mirror chunk arrives into the ring, which is then reversed and
    copied over the (already sent) chunk; a piece whose mirror lies in this
    rank's own shard is reversed locally."""
    rank = dist.get_rank(group)
    hi = lo + local.numel()
    a0, a1 = max(x, lo), min(z, hi)
    if a1 <= a0:
        return
    m0, m1 = x + z - a1, x + z - a0  # where my positions mirror to
    pieces = []  # (partner, my lo, my hi): my piece mirrors into the partner's shard
    for e in range(m0 // S, (m1 - 1) // S + 1):
        g0, g1 = max(m0, e * S), min(m1, (e + 1) * S)
        if g1 > g0:
            pieces.append((e, x + z - g1, x + z - g0))
    # every rank takes its pairs in one global order: no wait cycle
    for e, p0, p1 in sorted(pieces, key=lambda t: (min(t[0], rank), max(t[0], rank))):
        if e == rank:
            ops.reverse(local[p0 - lo:p1 - lo])  # symmetric about the centre
            _sync(local)
            continue
        # chunks pair mirror to mirror: the lower rank walks up, the higher down
        length, W = p1 - p0, ring.numel()
        for k in range(0, length, W):
            w = min(W, length - k)
            c0 = p0 + k if rank < e else p1 - k - w
            mine = local[c0 - lo:c0 - lo + w]
            buf = ring[:w]
            _exchange([(e, mine)], [(e, buf)], group)
            ops.reverse(buf)
            mine.copy_(buf)
            _sync(local)


def _rotate_range(local, lo, S, x, y, z, ops, group, ring) -> None:
    """Left-rotate the global range [x, z) so [y, z) comes first (strong.rotate,
    strong.py:85-95, by triple reversal)."""
    if x >= y or y >= z:
        return
    _reverse_range(local, lo, S, x, y, ops, group, ring)
    _reverse_range(local, lo, S, y, z, ops, group, ring)
    _reverse_range(local, lo, S, x, z, ops, group, ring)


def merge_interleave_plan(cr: list[int], q: list[int], world: int):
    """The rotations (level by level) that turn A_0..A_{G-1} B_0..B_{G-1}
    into A_0 B_0 .. A_{G-1} B_{G-1}, with A_d = A[cr[d]:cr[d+1]) and
    B_d = B[q[d] - cr[d] : q[d+1] - cr[d+1]) (q[d] = first output position of
    shard d).  Each entry (x, y, z): rotate [x, z) so that [y, z) comes
    first; the entries of one level touch disjoint groups of shards."""
    levels = []
    todo = [(0, world)]
    while todo:
        level, nxt = [], []
        for r0, r1 in todo:
            if r1 - r0 < 2:
                continue
            h = (r0 + r1) // 2
            # the group's range [q[r0], q[r1]) holds A_r0..A_{r1-1} B_r0..B_{r1-1};
            # bring B_r0..B_{h-1} in front of A_h..A_{r1-1}
            x = q[r0] + (cr[h] - cr[r0])                      # start of A_h
            y = q[r0] + (cr[r1] - cr[r0])                     # start of B_r0
            z = y + (q[h] - cr[h]) - (q[r0] - cr[r0])         # end of B_{h-1}
            level.append((x, y, z))
            nxt += [(r0, h), (h, r1)]
        if level:
            levels.append(level)
        todo = nxt
    return levels


def sharded_merge(local: torch.Tensor, n_global: int, split: int, ops: LocalOps,
                  group=None, wave_words: int = WAVE_WORDS) -> None:
    """Merge the sorted runs g[0:split) and g[split:n) of the sharded array
    in place (global output sorted, ties from the first run)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_bounds(n_global, world, rank)
    S = shard_bounds(n_global, world, 0)[1]
    qs = [min(d * S, n_global) for d in range(world + 1)]
    cr = merge_coranks(local, lo, n_global, split, qs, group)
    ring = torch.empty(max(1, min(wave_words, S)), dtype=local.dtype, device=local.device)
    for level in merge_interleave_plan(cr, qs, world):
        for x, y, z in level:
            _rotate_range(local, lo, S, x, y, z, ops, group, ring)
    # my shard now holds [A_rank | B_rank]
    ops.merge(local, cr[rank + 1] - cr[rank])
    _sync(local)
