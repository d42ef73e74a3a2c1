"""List contraction and list ranking on the GPU deterministic-reservations
engine (reference ``contraction.py:79-365``).

Same names, arguments and round structure as the reference: per round the
active prefix (failures of the previous round in order, then fresh ids
ascending, b(n) in all) is checked for local priority minima among active
neighbours, which splice out (``csrc/contraction.cu``).  ``RoundStats``
(rounds, committed-per-round) and ``trace`` equal the reference's; list
ranking finishes with in-place dependence waves over the contraction forest.
Tree contraction (``contraction.py:368-559``) runs its whole round loop on
the device (``csrc/tree.cu``): the frontier ring, the sweep cursor, the
active list, the active-id set and the rake-parent map live in the charged
workspace, and per round the host reads a few counts; rounds, traces,
roots and folded values equal the reference's.

Arrays may be numpy (host: copied to the device and back in place) or torch
CUDA tensors (processed in place on the current stream).  Validation
(``validate_linked_list``) is the reference's host-side input check.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .detres import RoundStats
from .runtime import EpsilonConfig, Rng, Words, alloc, as_words, release

__all__ = ["LinkedList", "BinaryTree", "make_priorities", "validate_linked_list",
           "validate_binary_tree", "list_contract", "list_rank", "tree_contract"]

DEFAULT_BUDGET = EpsilonConfig(epsilon=0.5)
NIL = (1 << 64) - 1
NIL32 = (1 << 32) - 1
_NILW = np.uint64(NIL)


@dataclass
class LinkedList:
    """Doubly-linked chains over index arrays; NIL terminates both ends
    (contraction.py:45-59)."""

    next: object
    prev: object

    def __post_init__(self) -> None:
        as_words(self.next)
        as_words(self.prev)
        if len(self.next) != len(self.prev):
            raise ValueError("next/prev length mismatch")

    def __len__(self) -> int:
        return len(self.next)


@dataclass
class BinaryTree:
    """Rooted forest of binary trees; internal nodes have exactly two children
    (contraction.py:62-76)."""

    parent: object
    left: object
    right: object

    def __post_init__(self) -> None:
        for arr in (self.parent, self.left, self.right):
            as_words(arr)
        if not len(self.parent) == len(self.left) == len(self.right):
            raise ValueError("parent/left/right length mismatch")

    def __len__(self) -> int:
        return len(self.parent)


def make_priorities(n: int, rng: Rng) -> np.ndarray:
    """Distinct random priorities: a random permutation of 0..n-1 made by the
    GPU permutation at the reference's derived seed (contraction.py:79-90)."""
    from .relaxed import make_swap_sequence, random_permutation

    p = np.arange(n, dtype=np.uint64)
    if n > 1:
        random_permutation(p, make_swap_sequence(n, rng.derive(0x707269)))
    return p


def _host(x) -> np.ndarray:
    if isinstance(x, np.ndarray):
        return x
    return x.detach().cpu().numpy().view(np.uint64)


def validate_linked_list(lst: LinkedList, deep: bool = True) -> None:
    """Reject malformed lists: dangling or non-inverse links, or cycles
    (contraction.py:96-127; host-side input check)."""
    n = len(lst)
    nxt, prv = _host(lst.next), _host(lst.prev)
    for arr, name in ((nxt, "next"), (prv, "prev")):
        live = arr != _NILW
        if bool(np.any(arr[live] >= np.uint64(n))):
            raise ValueError(f"{name} pointer out of range")
    ids = np.flatnonzero(nxt != _NILW)
    if bool(np.any(prv[nxt[ids]] != ids.astype(np.uint64))):
        raise ValueError("prev/next are not mutually inverse")
    ids = np.flatnonzero(prv != _NILW)
    if bool(np.any(nxt[prv[ids]] != ids.astype(np.uint64))):
        raise ValueError("prev/next are not mutually inverse")
    if not deep:
        return
    cur = np.flatnonzero(prv == _NILW).astype(np.uint64)
    seen = steps = 0
    while len(cur):
        seen += len(cur)
        cur = nxt[cur]
        cur = cur[cur != _NILW]
        steps += 1
        if steps > n + 1:
            break
    if seen != n:
        raise ValueError("list contains a cycle")


def validate_binary_tree(tree: BinaryTree, deep: bool = True) -> None:
    """contraction.py:130-165 (host-side input check)."""
    n = len(tree)
    pa, lf, rt = _host(tree.parent), _host(tree.left), _host(tree.right)
    for arr, name in ((pa, "parent"), (lf, "left"), (rt, "right")):
        live = arr != _NILW
        if bool(np.any(arr[live] >= np.uint64(n))):
            raise ValueError(f"{name} pointer out of range")
    if bool(np.any((lf == _NILW) != (rt == _NILW))):
        raise ValueError("internal nodes must have exactly two children")
    for child in (lf, rt):
        ids = np.flatnonzero(child != _NILW)
        if bool(np.any(pa[child[ids]] != ids.astype(np.uint64))):
            raise ValueError("child/parent links inconsistent")
    ids = np.flatnonzero(pa != _NILW).astype(np.uint64)
    if len(ids):
        up = pa[ids]
        if bool(np.any((lf[up] != ids) & (rt[up] != ids))):
            raise ValueError("child/parent links inconsistent")
    if not deep:
        return
    frontier = np.flatnonzero(pa == _NILW).astype(np.uint64)
    seen = steps = 0
    while len(frontier):
        seen += len(frontier)
        kids = np.concatenate([lf[frontier], rt[frontier]])
        frontier = kids[kids != _NILW]
        steps += 1
        if steps > n + 1:
            break
    if seen != n:
        raise ValueError("tree contains a cycle or unreachable nodes")


_SCAN_BLOCK = 4096
_COMBINE = {np.add: 0, np.maximum: 1, np.minimum: 2, np.bitwise_xor: 3}


def tree_contract(tree: BinaryTree, p, values, budget: EpsilonConfig = DEFAULT_BUDGET,
                  combine=np.add, trace: list | None = None, validate: bool = False,
                  debug: bool = False):
    """Contract the forest (rake leaves into parents, compress unary nodes
    into their child; contraction.py:528-559); returns ({root id: folded
    value}, stats).  ``values`` is folded in place; ``combine`` is one of
    np.add (default, mod 2^64), np.maximum, np.minimum, np.bitwise_xor."""
    import torch

    as_words(p)
    as_words(values)
    n = len(tree)
    if len(p) != n or len(values) != n:
        raise ValueError("priorities/values length mismatch")
    if combine not in _COMBINE:
        raise TypeError("combine must be np.add, np.maximum, np.minimum or np.bitwise_xor "
                        "(the device folds with atomics)")
    if validate:
        validate_binary_tree(tree)
    if n == 0:
        return {}, RoundStats()
    if n >= NIL32:
        raise ValueError("tree contraction supports fewer than 2^32 - 1 nodes")
    op = _COMBINE[combine]
    host_mode = isinstance(tree.parent, np.ndarray)
    if host_mode:
        dev = torch.cuda.current_device()
        pa, lf, rt = (torch.from_numpy(x.view(np.int64)).cuda()
                      for x in (tree.parent, tree.left, tree.right))
    else:
        dev = as_words(tree.parent, _wrap=True).device
        pa, lf, rt = tree.parent, tree.left, tree.right
    cuda = f"cuda:{dev}"

    def to_dev(x):
        return (torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).to(cuda)
                if isinstance(x, np.ndarray) else x)

    pt, vt = to_dev(p), to_dev(values)
    lib = _lib.load()
    prefix = budget.prefix_words(n)
    # the whole round loop on the device (csrc/tree.cu): frontier ring,
    # sweep cursor, active list, active-id set and rake-parent map in the
    # charged workspace; per round the host reads a few counts
    cap = max(16, 4 * n // max(prefix, 1) + 4096)
    counts = np.zeros(cap, dtype=np.uint64)
    tr = np.zeros(n if trace is not None else 0, dtype=np.uint64)
    roots_buf = np.zeros(2 * n, dtype=np.uint64)
    rounds, nroots, viol = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev).cuda_stream
        wb = lib.pip_tree_contract_workspace_bytes(n, prefix)
        buf = alloc(wb, dev)
        try:
            rc = lib.pip_tree_contract_u64(
                pa.data_ptr(), lf.data_ptr(), rt.data_ptr(), pt.data_ptr(), vt.data_ptr(), n, prefix, op,
                1 if debug else 0, counts.ctypes.data, cap, C.byref(rounds),
                tr.ctypes.data if len(tr) else None, roots_buf.ctypes.data, C.byref(nroots),
                C.byref(viol), buf.ptr, wb, st)
            if rc == _lib.PIP_ERR_TABLE:
                raise RuntimeError("tree contraction frontier overflow")
            _lib.check(rc, "tree contraction")
        finally:
            release(buf)
    stats = RoundStats()
    stats.rounds = int(rounds.value)
    stats.committed_per_round = [int(x) for x in counts[:min(stats.rounds, cap)]]
    if trace is not None:
        pos = 0
        for c in stats.committed_per_round:
            trace.append(tr[pos:pos + c].copy())
            pos += c
    k = int(nroots.value)
    roots = {int(r): int(v) for r, v in zip(roots_buf[0:2 * k:2].tolist(), roots_buf[1:2 * k:2].tolist())}
    if host_mode:
        tree.parent[:] = pa.cpu().numpy().view(np.uint64)
        tree.left[:] = lf.cpu().numpy().view(np.uint64)
        tree.right[:] = rt.cpu().numpy().view(np.uint64)
    if isinstance(values, np.ndarray):
        values[:] = vt.cpu().numpy().view(np.uint64)
    if debug and int(viol.value):
        raise AssertionError(f"{int(viol.value)} parent-child pairs contracted together")
    return roots, stats


def _run(lst: LinkedList, p, rank: bool, budget: EpsilonConfig, trace, on_splice):
    import torch

    n = len(lst)
    host_mode = isinstance(lst.next, np.ndarray)
    if host_mode != isinstance(lst.prev, np.ndarray):
        raise TypeError("next and prev must both be numpy arrays or both device tensors")
    wn: Words = as_words(lst.next, _wrap=True)
    if host_mode:
        dn = torch.from_numpy(lst.next.view(np.int64)).cuda()
        dp = torch.from_numpy(lst.prev.view(np.int64)).cuda()
        dev = torch.cuda.current_device()
    else:
        dn, dp = lst.next, lst.prev
        dev = wn.device
    if isinstance(p, np.ndarray):
        pt = torch.from_numpy(np.ascontiguousarray(p).view(np.int64)).to(f"cuda:{dev}")
    else:
        pt = p
    prefix = budget.prefix_words(n)
    lib = _lib.load()
    cap = max(16, 2 * n // max(prefix, 1) + 4096)
    counts = (C.c_uint64 * cap)()
    rounds = C.c_uint64(0)
    tr = np.zeros(n if (trace is not None or on_splice is not None) else 0, dtype=np.uint64)
    sp = np.zeros(3 * n if on_splice is not None else 0, dtype=np.uint64)
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev).cuda_stream
        wb = lib.pip_list_contract_workspace_bytes(n, prefix, 1 if rank else 0)
        buf = alloc(wb, dev)
        try:
            _lib.check(lib.pip_list_contract_u64(
                dn.data_ptr(), dp.data_ptr(), pt.data_ptr(), n, prefix, 1 if rank else 0, counts,
                cap, C.byref(rounds), tr.ctypes.data if len(tr) else None,
                sp.ctypes.data if len(sp) else None, buf.ptr, wb, st), "list contraction")
        finally:
            release(buf)
    if host_mode:
        lst.next[:] = dn.cpu().numpy().view(np.uint64)
        lst.prev[:] = dp.cpu().numpy().view(np.uint64)
    stats = RoundStats()
    stats.rounds = int(rounds.value)
    stats.committed_per_round = [int(counts[i]) for i in range(min(stats.rounds, cap))]
    pos = 0
    for c in stats.committed_per_round:
        if trace is not None:
            trace.append(tr[pos:pos + c].copy())
        if on_splice is not None and c:
            t = sp[3 * pos:3 * (pos + c)].reshape(c, 3)
            on_splice(t[:, 0].copy(), t[:, 1].copy(), t[:, 2].copy())
        pos += c
    return stats


def list_contract(lst: LinkedList, p, on_splice=None, budget: EpsilonConfig = DEFAULT_BUDGET,
                  trace: list | None = None, validate: bool = False) -> RoundStats:
    """Splice out every element; per round the active-prefix local minima go
    (contraction.py:264-289).  Afterwards each element's (prev, next) slots
    hold the neighbours it saw when spliced; ``on_splice(ids, prevs, nexts)``
    observes each round's batch."""
    as_words(p)
    n = len(lst)
    if len(p) != n:
        raise ValueError("priorities length mismatch")
    if validate:
        validate_linked_list(lst)
    if n == 0:
        return RoundStats()
    return _run(lst, p, False, budget, trace, on_splice)


def list_rank(lst: LinkedList, p, budget: EpsilonConfig = DEFAULT_BUDGET,
              trace: list | None = None, validate: bool = False,
              stats_sink: list | None = None):
    """Rank every element within its chain, in place over the list storage
    (contraction.py:323-365): afterwards ``lst.prev`` holds the 0-based ranks
    (and is returned) and ``lst.next`` bookkeeping marks."""
    as_words(p)
    n = len(lst)
    if len(p) != n:
        raise ValueError("priorities length mismatch")
    if n >= NIL32:
        raise ValueError("list ranking supports fewer than 2^32 - 1 elements")
    if validate:
        validate_linked_list(lst)
    if n == 0:
        return lst.prev
    stats = _run(lst, p, True, budget, trace, None)
    if stats_sink is not None:
        stats_sink.append(stats)
    return lst.prev
