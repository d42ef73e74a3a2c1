"""Strong (zero-heap) in-place operations on the GPU — drop-in for
``pipal.strong`` (reference strong.py).

Signatures, return values and errors follow the reference:
  scan(a, op=None, identity=0, base=256) -> ScanResult      strong.py:151-166
  scan_blocked(a, op=None, identity=0, block=256)           strong.py:169-236
  reduce(a, op=None, identity=0) -> int                     strong.py:43-64
  rotate(a, o)                                              strong.py:85-95
  filter_kway(a, pred, n=None) -> int                       strong.py:283-349
  merge_strong(a, split, debug=False)                       strong.py:496-522
``a`` is either a numpy uint64 array (copied through the device by the
library's host-buffer entry points and written back in place) or a torch
CUDA tensor (uint64/int64, processed in place on the current stream).

Zero heap: nothing here charges the space meter.  Scan, filter, reduce and
rotate use O(#CTAs) look-back scratch (the analogue of the reference's
O(log n) recursion stack); merge_strong additionally uses O(n / 8192) chunk
descriptors plus one 64 KiB chunk per SM of unmetered device scratch
("workspace").
"""
from __future__ import annotations

import ctypes as C
import os
import operator
from dataclasses import dataclass

import numpy as np

from . import _lib
from .pred import as_pred
from .runtime import M64, Words, as_words, scratch_for, small_device_words

__all__ = ["ScanResult", "scan", "scan_blocked", "scan_inclusive", "reduce", "rotate",
           "filter_kway", "partition_unstable", "quicksort_strong", "merge_strong"]

SCAN_BASE = 256


@dataclass
class ScanResult:
    array: object
    total: int


def _device_index() -> int:
    import torch

    return torch.cuda.current_device()


def _op_code(op):
    """Map the reference's `op` callables onto the kernel's element ops."""
    if op is None or op is operator.add:
        return _lib.OP_ADD
    if op is max:
        return _lib.OP_MAX
    if op is min:
        return _lib.OP_MIN
    if op is operator.xor or op is operator.ixor:
        return _lib.OP_XOR
    raise TypeError("GPU scan supports op in {None, operator.add, max, min, operator.xor}; "
                    "arbitrary callables cannot run on the device")


def _identity_of(code: int) -> int:
    return M64 if code == _lib.OP_MIN else 0


def _scan_impl(a, op, identity, inclusive: bool) -> ScanResult:
    w: Words = as_words(a, _wrap=True)
    code = _op_code(op)
    n = w.n
    # reference: op=None always starts from 0 and reports `identity & M64`
    # for an empty array; a given op starts from `identity`
    init = 0 if op is None else int(identity) & M64
    if n == 0:
        return ScanResult(a, int(identity) & M64 if op is None else identity)
    lib = _lib.load()
    if w.is_device:
        import torch

        with torch.cuda.device(w.device):
            st = w.stream()
            sp, sb = scratch_for(w.device, st)
            tot = small_device_words(1, w.device)
            _lib.check(lib.pip_scan_u64(w.ptr, n, code, init, 1 if inclusive else 0, tot.data_ptr(),
                                        sp, sb, st), "scan")
            _lib.check_stall(sp, st, "scan")
            total = int(tot.item()) & M64
    else:
        out = C.c_uint64(0)
        _lib.check(lib.pip_scan_u64_host(w.ptr, n, code, init, 1 if inclusive else 0,
                                         C.byref(out), _device_index()), "scan")
        total = int(out.value)
    return ScanResult(a, total)


def scan(a, op=None, identity: int = 0, base: int = SCAN_BASE) -> ScanResult:
    """Exclusive in-place scan; returns the rewritten array and the total."""
    return _scan_impl(a, op, identity, inclusive=False)


def scan_blocked(a, op=None, identity: int = 0, block: int = SCAN_BASE) -> ScanResult:
    """Blocked scan (strong.py:169-236): same contract, bit-identical to scan."""
    return _scan_impl(a, op, identity, inclusive=False)


def scan_inclusive(a, op=None, identity: int = 0) -> ScanResult:
    """Inclusive in-place scan (BASELINE config 1): a[i] = x0 op ... op x_i.

    Equals the reference's exclusive scan shifted left by one with the total
    appended (``a[1:] ++ [total]``), i.e. ``np.cumsum`` for op=None.
    """
    return _scan_impl(a, op, identity, inclusive=True)


def reduce(a, op=None, identity: int = 0) -> int:
    """Fold the array with an associative op; the array is not modified."""
    w: Words = as_words(a, _wrap=True)
    code = _op_code(op)
    if w.n == 0:
        return identity & M64 if op is None else identity
    lib = _lib.load()
    if w.is_device:
        import torch

        with torch.cuda.device(w.device):
            st = w.stream()
            sp, sb = scratch_for(w.device, st)
            tot = small_device_words(1, w.device)
            _lib.check(lib.pip_reduce_u64(w.ptr, w.n, code, tot.data_ptr(), sp, sb, st), "reduce")
            _lib.check_stall(sp, st, "reduce")
            return int(tot.item()) & M64
    # host array: stream it through the device with a read-only scan copy
    import torch

    dev = torch.from_numpy(w.obj.view(np.int64)).cuda()
    return reduce(dev, op, identity)


def rotate(a, o: int) -> None:
    """Left-rotate in place: output[i] = input[(i + o) mod n] (triple reversal)."""
    w: Words = as_words(a, _wrap=True)
    n = w.n
    if not 0 <= o <= n:
        raise ValueError("offset must lie in [0, n]")
    if o == 0 or o == n or n < 2:
        return
    lib = _lib.load()
    if w.is_device:
        import torch

        with torch.cuda.device(w.device):
            st = w.stream()
            _lib.check(lib.pip_rotate_u64(w.ptr, n, o, None, 0, st), "rotate")
        return
    _via_device(w.obj, lambda t: rotate(t, o))


def _via_device(arr: np.ndarray, fn):
    """Run a device op on a host array: H2D, fn(tensor), D2H in place."""
    import torch

    t = torch.from_numpy(arr.view(np.int64)).cuda()
    r = fn(t)
    arr[:] = t.cpu().numpy().view(np.uint64)
    return r


def filter_kway(a, pred, n: int | None = None) -> int:
    """Stable in-place filter: kept elements end up in a[0:m); returns m.

    ``pred`` must be a :class:`~paper_2103_01216_b200.pred.Pred`.  Only the
    first ``n`` words are filtered when ``n`` is given (strong.py:283-292).
    """
    w: Words = as_words(a, _wrap=True)
    p = as_pred(pred)
    n = w.n if n is None else int(n)
    if n < 0 or n > w.n:
        raise ValueError("n out of range")
    if n == 0:
        return 0
    lib = _lib.load()
    desc = p.descriptor()
    if w.is_device:
        import torch

        with torch.cuda.device(w.device):
            st = w.stream()
            sp, sb = scratch_for(w.device, st)
            m = small_device_words(1, w.device)
            _lib.check(lib.pip_filter_u64(w.ptr, n, C.byref(desc), m.data_ptr(), sp, sb, st),
                       "filter")
            _lib.check_stall(sp, st, "filter")
            return int(m.item())
    out = C.c_uint64(0)
    _lib.check(lib.pip_filter_u64_host(w.ptr, n, C.byref(desc), C.byref(out), _device_index()),
               "filter")
    return int(out.value)


def _partition_impl(a, pred, n: int | None, meter_workspace: bool) -> int:
    w: Words = as_words(a, _wrap=True)
    p = as_pred(pred)
    n = w.n if n is None else int(n)
    if n < 0 or n > w.n:
        raise ValueError("n out of range")
    if n == 0:
        return 0
    lib = _lib.load()
    desc = p.descriptor()
    wb = lib.pip_partition_workspace_bytes(n)
    if not w.is_device:
        out = C.c_uint64(0)
        if meter_workspace:
            from .runtime import charge, uncharge

            _charged = charge((wb + 7) // 8)
        try:
            _lib.check(lib.pip_partition_u64_host(w.ptr, n, C.byref(desc), C.byref(out),
                                                  _device_index()), "partition")
        finally:
            if meter_workspace:
                uncharge((wb + 7) // 8, _charged)
        return int(out.value)
    import torch

    from .runtime import alloc, release

    with torch.cuda.device(w.device):
        st = w.stream()
        if meter_workspace:
            buf = alloc(wb, w.device)
            ptr, keep = buf.ptr, buf
        else:
            keep = torch.empty(max(wb, 16), dtype=torch.uint8, device=f"cuda:{w.device}")
            ptr, buf = keep.data_ptr(), None
        try:
            m = small_device_words(1, w.device)
            _lib.check(lib.pip_partition_u64(w.ptr, n, C.byref(desc), m.data_ptr(), ptr, wb, st),
                       "partition")
            return int(m.item())
        finally:
            if buf is not None:
                release(buf)
            del keep


def partition_unstable(a, pred, n: int | None = None) -> int:
    """Unstable in-place partition (strong.py:394-419): the words with
    ``pred`` true end up in a[0:m), the others in a[m:n); returns m.

    ``pred`` is a :class:`~paper_2103_01216_b200.pred.Pred`.  The GPU swaps
    the false words left of m with the true words right of m by rank (one
    count pass, one swap pass); its O(n/4096) descriptors are device scratch,
    like the reference's unmetered recursion space.
    """
    return _partition_impl(a, pred, n, meter_workspace=False)


# leaves: sorted by one grid-wide bitonic network (pip_sort_segments_grid_u64)
QS_LEAF = int(os.environ.get("PIP_QS_LEAF", 1 << 22))


def _quicksort_impl(a, rng, salt_of, meter_workspace: bool) -> None:
    """Quicksort over the GPU partition (strong.py:422-454, relaxed.py:347-371):
    segments longer than QS_LEAF words are split around a pivot picked with
    the reference's rule (a[lo + rng.word(((lo << 21) ^ hi) + salt) % (hi -
    lo)]) by two partitions (< pivot, == pivot); the leaves are sorted by one
    launch.  The output is the sorted array whatever the pivots."""
    import torch

    w: Words = as_words(a, _wrap=True)
    n = w.n
    if n < 2:
        return None
    if not w.is_device:
        return _via_device(w.obj, lambda t: _quicksort_impl(t, rng, salt_of, meter_workspace))
    from .pred import eq, lt
    from .runtime import alloc, release

    lib = _lib.load()
    with torch.cuda.device(w.device):
        st = w.stream()
        wb = lib.pip_partition_workspace_bytes(n)
        if meter_workspace:
            buf = alloc(wb, w.device)
            ws_ptr, keep = buf.ptr, buf
        else:
            keep = torch.empty(max(wb, 16), dtype=torch.uint8, device=f"cuda:{w.device}")
            ws_ptr, buf = keep.data_ptr(), None
        try:
            words = w.obj.view(torch.int64) if w.obj.dtype != torch.int64 else w.obj
            dev = f"cuda:{w.device}"

            def part_all(los, lens, pvs, kind, mbuf) -> list[int]:
                # every partition of the level in one call (they share the
                # workspace stream-ordered); one read of all counts
                k = len(los)
                arr = (C.c_uint64 * k)
                _lib.check(lib.pip_partition_segments_u64(w.ptr, arr(*los), arr(*lens), arr(*pvs),
                                                          kind, mbuf.data_ptr(), k, ws_ptr, wb, st),
                           "partition")
                return mbuf.cpu().tolist()

            leaves_lo: list[int] = []
            leaves_len: list[int] = []
            # Level-batched recursion: the segments of one depth are disjoint,
            # so their pivots are gathered with one read and their partitions
            # queued back to back -- three host syncs per level, not per
            # segment.  Pivot rule and per-segment depth as in the sequential
            # recursion (strong.py:431-454).
            level = [(0, n, 0)]
            while level:
                big = []
                for lo, hi, depth in level:
                    if hi - lo > QS_LEAF:
                        big.append((lo, hi, depth))
                    elif hi - lo > 1:
                        leaves_lo.append(lo)
                        leaves_len.append(hi - lo)
                if not big:
                    break
                idx = [lo + rng.word(((lo << 21) ^ hi) + salt_of(depth)) % (hi - lo)
                       for lo, hi, depth in big]
                pvs = [int(v) & M64 for v in
                       words[torch.tensor(idx, dtype=torch.int64, device=dev)].cpu().tolist()]
                mbuf = torch.empty(len(big), dtype=torch.int64, device=dev)
                less = part_all([lo for lo, _, _ in big], [hi - lo for lo, hi, _ in big], pvs,
                                lt(0).descriptor().kind, mbuf)
                equal = part_all([lo + le for (lo, _, _), le in zip(big, less)],
                                 [hi - lo - le for (lo, hi, _), le in zip(big, less)], pvs,
                                 eq(0).descriptor().kind, mbuf)
                level = []
                for (lo, hi, depth), le, eqn in zip(big, less, equal):
                    level.append((lo, lo + le, depth + 1))
                    level.append((lo + le + eqn, hi, depth + 1))
            if leaves_lo:
                slo = torch.tensor(leaves_lo, dtype=torch.int64, device=dev)
                sln = torch.tensor(leaves_len, dtype=torch.int32, device=dev)
                _lib.check(lib.pip_sort_segments_grid_u64(w.ptr, slo.data_ptr(), sln.data_ptr(),
                                                          len(leaves_lo), max(leaves_len), st),
                           "sort")
                torch.cuda.current_stream(w.device).synchronize()
        finally:
            if buf is not None:
                release(buf)
            del keep
    return None


def quicksort_strong(a, rng) -> None:
    """In-place quicksort over the unstable partition (strong.py:422-454).

    ``rng`` is a :class:`~paper_2103_01216_b200.runtime.Rng`; pivots follow
    the reference's rule (its depth-cap restarts only change pivots, never
    the sorted output).  Leaves of <= 2^22 words (``PIP_QS_LEAF``) are sorted on the
    GPU by one grid-wide bitonic network (the reference's base case is
    ``a[lo:hi].sort()``).
    """
    _quicksort_impl(a, rng, lambda depth: 0, meter_workspace=False)


def _merge_impl(a, split: int, debug: bool, budget_words: int, meter_workspace: bool) -> None:
    from .runtime import alloc, release

    w: Words = as_words(a, _wrap=True)
    n = w.n
    if not 0 <= split <= n:
        raise ValueError("split out of range")
    lib = _lib.load()
    if not w.is_device:
        if debug:
            return _via_device(w.obj, lambda t: _merge_impl(t, split, debug, budget_words,
                                                             meter_workspace))
        if split == 0 or split == n or n < 2:
            return None
        # the streamed host merge's auxiliary device memory is its output
        # ring (the device copy of the array is staging, as on every host
        # path); that ring is what a relaxed call charges
        wb = lib.pip_merge_host_workspace_bytes(n, split, budget_words)
        words = (wb + 7) // 8
        if meter_workspace:
            from .runtime import charge, uncharge

            _charged = charge(words)
            try:
                _lib.check(lib.pip_merge_u64_host(w.ptr, n, split, budget_words, _device_index()),
                           "merge")
            finally:
                uncharge(words, _charged)
        else:
            _lib.check(lib.pip_merge_u64_host(w.ptr, n, split, budget_words, _device_index()),
                       "merge")
        return None
    import torch

    with torch.cuda.device(w.device):
        st = w.stream()
        sp, sb = scratch_for(w.device, st)
        wb = lib.pip_merge_workspace_bytes(n, split, budget_words)
        if meter_workspace:
            buf = alloc(wb, w.device)
            ptr, keep = buf.ptr, buf
        else:
            keep = torch.empty(max(wb, 16), dtype=torch.uint8, device=f"cuda:{w.device}")
            ptr, buf = keep.data_ptr(), None
        try:
            _lib.check(lib.pip_merge_u64(w.ptr, n, split, 1 if debug else 0, ptr if wb else None,
                                         wb, sp, sb, st), "merge")
        finally:
            if buf is not None:
                release(buf)
            del keep
    return None


def merge_strong(a, split: int, debug: bool = False) -> None:
    """In-place merge of the sorted runs a[0:split) and a[split:n)."""
    _merge_impl(a, split, debug, 0, meter_workspace=False)
