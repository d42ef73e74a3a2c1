"""Relaxed in-place operations on the GPU — drop-in for ``pipal.relaxed``
(reference relaxed.py).

  make_swap_sequence(n, rng) / validate_swap_sequence(h)      relaxed.py:47-58
  random_permutation(a, h, variant="final", budget, trace, debug)
                                              -> RoundStats   relaxed.py:220-251
  decompose_driver(n, budget_words, step, trace)              relaxed.py:257-278
  filter_relaxed(a, pred, budget, stats_sink) -> int          relaxed.py:284-309
  merge_relaxed(a, split, budget, debug)                      relaxed.py:579-612

Every charged buffer is DEVICE workspace, metered in 64-bit words through
the active ``SpaceMeter`` exactly like the reference's runtime.alloc.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .detres import LivelockError, RoundStats
from .pred import as_pred
from .runtime import (
    WORD,
    EpsilonConfig,
    Words,
    alloc,
    as_words,
    release,
    scratch_for,
    small_device_words,
)
from .strong import _merge_impl, _quicksort_impl

__all__ = ["RP_VARIANTS", "DEFAULT_BUDGET", "make_swap_sequence", "validate_swap_sequence",
           "random_permutation", "decompose_driver", "filter_relaxed", "partition_relaxed",
           "quicksort_relaxed", "merge_relaxed"]

DEFAULT_BUDGET = EpsilonConfig(epsilon=0.5)
RP_VARIANTS = ("naive", "flat", "oneres", "final")
_VARIANT_CODE = {"naive": _lib.RP_NAIVE, "flat": _lib.RP_FLAT, "oneres": _lib.RP_ONERES,
                 "final": _lib.RP_FINAL}
_ROUNDS_CAP = 1 << 22


def make_swap_sequence(n: int, rng) -> np.ndarray:
    """H with H[i] uniform over [0, i] (0-indexed) — relaxed.py:47-52."""
    if n == 0:
        return np.empty(0, dtype=WORD)
    words = rng.words(0, n)
    return words % (np.arange(n, dtype=WORD) + WORD(1))


def validate_swap_sequence(h) -> None:
    """ValueError unless H[i] <= i for all i (relaxed.py:55-58); on device."""
    w: Words = as_words(h, _wrap=True)
    if w.n == 0:
        return
    if not w.is_device:
        import torch

        validate_swap_sequence(torch.from_numpy(w.obj.view(np.int64)).cuda())
        return
    import torch

    lib = _lib.load()
    with torch.cuda.device(w.device):
        st = w.stream()
        sp, sb = scratch_for(w.device, st)
        _lib.check(lib.pip_validate_swaps_u64(w.ptr, w.n, None, sp, sb, st), "validate")


def random_permutation(a, h, variant: str = "final", budget: EpsilonConfig = DEFAULT_BUDGET,
                       trace: list | None = None, debug: bool = False) -> RoundStats:
    """Apply the swap sequence in parallel rounds, in place.

    The output equals the sequential shuffle with the same ``h``
    (baselines.seq_knuth_shuffle); rounds, committed-per-round, trace and
    peak_table_load equal the reference's because the GPU engine keeps its
    round structure (see csrc/rp.cu).
    """
    wa: Words = as_words(a, _wrap=True)
    wh: Words = as_words(h, _wrap=True)
    if wh.n != wa.n:
        raise ValueError("swap sequence length must match the array")
    if variant not in RP_VARIANTS:
        # the reference validates H first (relaxed.py:233), then the variant
        validate_swap_sequence(h)
        raise ValueError(f"unknown variant {variant!r}")
    n = wa.n
    if n == 0:
        return RoundStats()
    import torch

    if not wa.is_device or not wh.is_device:
        da = torch.from_numpy(wa.to_numpy().view(np.int64)).cuda() if not wa.is_device else wa.obj
        dh = torch.from_numpy(wh.to_numpy().view(np.int64)).cuda() if not wh.is_device else wh.obj
        stats = random_permutation(da, dh, variant, budget, trace, debug)
        if not wa.is_device:
            wa.obj[:] = da.cpu().numpy().view(np.uint64)
        return stats
    if wa.device != wh.device:
        raise ValueError("a and h must live on the same device")
    lib = _lib.load()
    prefix = budget.prefix_words(n)
    code = _VARIANT_CODE[variant]
    with torch.cuda.device(wa.device):
        st = wa.stream()
        wb = lib.pip_rp_workspace_bytes(n, prefix, code)
        ws = alloc(wb, wa.device)
        cap = min(n, _ROUNDS_CAP)
        counts = np.zeros(max(cap, 1), dtype=np.uint64)
        tbuf = small_device_words(n, wa.device) if trace is not None else None
        stats = _lib.PipRpStats()
        try:
            rc = lib.pip_random_permutation_u64(
                wa.ptr, wh.ptr, n, prefix, code, 1 if debug else 0,
                counts.ctypes.data, cap, tbuf.data_ptr() if tbuf is not None else None,
                ws.ptr, wb, C.byref(stats), st)
            if rc == _lib.PIP_ERR_DEBUG_SWEEP:
                raise AssertionError("debug sweep: reservation slots not clean after a round")
            _lib.check(rc, "random_permutation")
        finally:
            release(ws)
    rounds = int(stats.rounds)
    if rounds > cap:
        raise RuntimeError(f"{rounds} rounds exceed the per-round record capacity {cap}")
    per_round = [int(x) for x in counts[:rounds]]
    out = RoundStats(rounds=rounds, committed_per_round=per_round,
                     peak_table_load=(int(stats.peak_table_count) / int(stats.table_capacity))
                     if stats.table_capacity else 0.0)
    if trace is not None and rounds:
        tr = tbuf[: int(stats.total_committed)].cpu().numpy().view(np.uint64)
        pos = 0
        for c in per_round:
            trace.append(tr[pos:pos + c].copy())
            pos += c
    return out


def decompose_driver(n: int, budget_words: int, step, trace: list | None = None) -> RoundStats:
    """Iterate ``step(count_hint) -> retired`` until the problem is empty
    (relaxed.py:257-278; host-side control logic, unchanged)."""
    if budget_words < 1:
        raise ValueError("budget must be >= 1")
    stats = RoundStats()
    remaining = n
    zero_rounds = 0
    while remaining > 0:
        done = int(step(min(budget_words, remaining)))
        stats.rounds += 1
        stats.committed_per_round.append(done)
        if trace is not None:
            trace.append(done)
        if done <= 0:
            zero_rounds += 1
            if zero_rounds >= 64:
                raise LivelockError("step retired nothing for 64 rounds")
        else:
            zero_rounds = 0
        remaining -= done
    return stats


def _relaxed_rounds(a, pred, budget: EpsilonConfig, stats_sink, kind: str) -> int:
    """The reference's prefix rounds (decompose_driver over b(n)-word blocks,
    relaxed.py:284-344) run on the device, one block per round:

      filter:    the block is filtered in place (stable, pip_filter_u64) and
                 its kept words move down to a[m:] (pip_move_u64, one pass);
      partition: the block is partitioned in place (pip_partition_u64), then
                 the first d = min(#true, #false so far) false words of
                 a[m:pos) and the last d true words of the block swap places
                 through a charged d-word buffer (the reference's displaced
                 words, relaxed.py:326-335), so a[0:m') is all true and
                 a[m':pos') all false.

    So the rounds, their retired counts and the b(n)-word buffer are the
    reference's, not a restatement of them; the word order inside the false
    region may differ from the reference's (its contract leaves it free).
    """
    import torch

    w: Words = as_words(a, _wrap=True)
    p = as_pred(pred)
    n = w.n
    if n == 0:
        return 0
    if not w.is_device:
        t = torch.from_numpy(w.obj.view(np.int64)).cuda()
        m = _relaxed_rounds(t, pred, budget, stats_sink, kind)
        w.obj[:] = t.cpu().numpy().view(np.uint64)
        return m
    b = budget.prefix_words(n)
    lib = _lib.load()
    desc = p.descriptor()
    words = w.obj.view(torch.int64) if w.obj.dtype != torch.int64 else w.obj
    state = {"m": 0, "pos": 0}
    with torch.cuda.device(w.device):
        st = w.stream()
        sp, sb = scratch_for(w.device, st)
        cnt = small_device_words(1, w.device)
        if kind == "partition":
            buf = alloc(8 * b, w.device)  # the reference's aux(b) (relaxed.py:320)
            tmp = buf.tensor[: 8 * b].view(torch.int64)
            wb = lib.pip_partition_workspace_bytes(b)
            pws = alloc(wb, w.device)  # the block partition's descriptors
        try:
            def step(hint: int) -> int:
                pos, m = state["pos"], state["m"]
                take = min(hint, n - pos)
                blk = w.ptr + 8 * pos
                if kind == "filter":
                    _lib.check(lib.pip_filter_u64(blk, take, C.byref(desc), cnt.data_ptr(), sp, sb,
                                                  st), "filter_relaxed")
                    _lib.check_stall(sp, st, "filter_relaxed")
                    k = int(cnt.item())
                    if k and m < pos:
                        _lib.check(lib.pip_move_u64(w.ptr, m, pos, k, sp, sb, st), "filter_relaxed")
                        _lib.check_stall(sp, st, "filter_relaxed")
                    state["m"] = m + k
                else:
                    _lib.check(lib.pip_partition_u64(blk, take, C.byref(desc), cnt.data_ptr(),
                                                     pws.ptr, wb, st), "partition_relaxed")
                    tc = int(cnt.item())
                    d = min(tc, pos - m)
                    if d:
                        x = words[m:m + d]                        # displaced false words
                        y = words[pos + tc - d:pos + tc]          # the block's last d true words
                        tmp[:d].copy_(x)
                        x.copy_(y)
                        y.copy_(tmp[:d])
                    state["m"] = m + tc
                state["pos"] = pos + take
                return take

            stats = decompose_driver(n, b, step)
        finally:
            if kind == "partition":
                release(pws)
                release(buf)
    if stats_sink is not None:
        stats_sink.append(stats)
    return state["m"]


def filter_relaxed(a, pred, budget: EpsilonConfig = DEFAULT_BUDGET,
                   stats_sink: list | None = None) -> int:
    """Stable filter, one b(n)-word block per round (relaxed.py:284-309):
    a[0:m) = the kept words in order; returns m; ``stats_sink`` receives the
    rounds the device actually ran (ceil(n / b) blocks)."""
    return _relaxed_rounds(a, pred, budget, stats_sink, "filter")


def partition_relaxed(a, pred, budget: EpsilonConfig = DEFAULT_BUDGET,
                      stats_sink: list | None = None) -> int:
    """Unstable partition, one b(n)-word block per round (relaxed.py:312-344):
    a[0:m) holds the words with ``pred`` true, a[m:n) the others (multiset
    preserved); returns m."""
    return _relaxed_rounds(a, pred, budget, stats_sink, "partition")


def quicksort_relaxed(a, rng, budget: EpsilonConfig = DEFAULT_BUDGET) -> None:
    """Quicksort over the relaxed partition (relaxed.py:347-371): segments run
    one at a time, so the charged footprint is one partition's descriptors
    (O(n/2048) words); pivots use the reference's rule with salt 0."""
    as_words(a, _wrap=True)
    _quicksort_impl(a, rng, lambda depth: 0, meter_workspace=True)


def merge_relaxed(a, split: int, budget: EpsilonConfig = DEFAULT_BUDGET,
                  debug: bool = False) -> None:
    """In-place merge of a[0:split) and a[split:n) within the budget b(n).

    The workspace (chunk descriptors + cut buffer for the chunk permutation)
    is sized from b(n) and charged to the active meter.
    """
    w: Words = as_words(a, _wrap=True)
    n = w.n
    if not 0 <= split <= n:
        raise ValueError("split out of range")
    b = budget.prefix_words(n) if n else 1
    _merge_impl(a, split, debug, max(int(b), 1), meter_workspace=True)
