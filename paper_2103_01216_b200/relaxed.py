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
from .strong import _merge_impl, _partition_impl, _quicksort_impl, filter_kway

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


def filter_relaxed(a, pred, budget: EpsilonConfig = DEFAULT_BUDGET,
                   stats_sink: list | None = None) -> int:
    """Stable filter with the reference's prefix-round contract.

    The GPU retires the whole array in one look-back pass with no buffer
    (0 charged words <= 8 b(n)); the returned m and a[0:m) equal the
    reference's, and ``stats_sink`` receives the round structure the
    reference reports (ceil(n / b) rounds of min(b, remaining) words).
    """
    w: Words = as_words(a, _wrap=True)
    as_pred(pred)
    n = w.n
    if n == 0:
        return 0
    b = budget.prefix_words(n)
    m = filter_kway(a, pred)
    if stats_sink is not None:
        st = RoundStats()
        rem = n
        while rem > 0:
            take = min(b, rem)
            st.rounds += 1
            st.committed_per_round.append(take)
            rem -= take
        stats_sink.append(st)
    return m


def partition_relaxed(a, pred, budget: EpsilonConfig = DEFAULT_BUDGET,
                      stats_sink: list | None = None) -> int:
    """Unstable partition with the reference's prefix-round contract
    (relaxed.py:312-344): a[0:m) holds the words with ``pred`` true, a[m:n)
    the others (multiset preserved); returns m.

    The GPU runs the swap partition of ``strong.partition_unstable`` once over
    the whole array; its O(n/4096) descriptor words are charged to the active
    meter (well under b(n)), and ``stats_sink`` receives the reference's
    round structure (ceil(n / b) rounds of min(b, remaining) words).
    """
    w = as_words(a, _wrap=True)
    as_pred(pred)
    n = w.n
    if n == 0:
        return 0
    b = budget.prefix_words(n)
    m = _partition_impl(a, pred, None, meter_workspace=True)
    if stats_sink is not None:
        st = RoundStats()
        rem = n
        while rem > 0:
            take = min(b, rem)
            st.rounds += 1
            st.committed_per_round.append(take)
            rem -= take
        stats_sink.append(st)
    return m


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
