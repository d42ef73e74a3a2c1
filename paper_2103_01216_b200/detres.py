"""Deterministic-reservations round engine and write-max reservation table
on the GPU — drop-in for ``pipal.detres`` (reference detres.py).

* :class:`ReservationTable` (detres.py:40-211): the open-addressed,
  linear-probed word->word write-max map, its key/value arrays in device
  memory (charged to the active meter: 2 x capacity words, as the
  reference's ``alloc``), batch updates by ``pip_rt_reserve_max_u64`` — the
  reference's probe-step algorithm reproduced step for step, so even the
  slot layout matches (csrc/detres.cu).  Keys/values may be numpy arrays
  (results come back as numpy) or CUDA tensors (results stay on the device).
* :func:`run_rounds` / :class:`RoundView` (detres.py:233-307): the round
  driver.  The active prefix (``ids``, int64) and the ``committed`` flags
  live in device memory (charged: prefix + ceil(prefix/8) words, as the
  reference's ``alloc`` / ``alloc_bool``); the phase callbacks receive CUDA
  tensor views and run device work on them; failures are packed in order
  by the device compaction (``pip_compact_by_mask_u64``, detres.py:303).
  The permutation (csrc/rp.cu) and list contraction (csrc/contraction.cu)
  run their whole round loop inside their own kernels; this engine is the
  generic one for other clients, as in the reference.
* :class:`RoundStats`, :class:`LivelockError`, ``LIVELOCK_ROUNDS``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .runtime import GOLDEN, WORD, alloc, release, scratch_for, small_device_words

__all__ = ["ReservationTable", "RoundStats", "RoundView", "run_rounds", "reserve_max",
           "LivelockError", "arange_source", "LIVELOCK_ROUNDS"]

LIVELOCK_ROUNDS = 64


class LivelockError(RuntimeError):
    """No iterate committed for LIVELOCK_ROUNDS consecutive rounds."""


def _torch():
    import torch

    return torch


def _device_words(x, device: int):
    """(int64 CUDA tensor of the words, was_numpy)."""
    torch = _torch()
    if isinstance(x, np.ndarray):
        a = np.ascontiguousarray(x, dtype=WORD)
        return torch.from_numpy(a.view(np.int64)).to(f"cuda:{device}"), True
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            return x.to(torch.int64).to(f"cuda:{device}"), True
        t = x.view(torch.int64) if x.dtype == torch.uint64 else x.to(torch.int64)
        return t.contiguous(), False
    return _device_words(np.asarray(x, dtype=WORD), device)


# ---------------------------------------------------------------------------
# Reservation table

class ReservationTable:
    """Open-addressed, linear-probed word->word map with write-max semantics
    (detres.py:40-211), held in device memory.

    Capacity is rounded up to a power of two (minimum 8); the caller keeps
    the load factor at or below one half.  ``reserve_max`` applies, per key,
    the maximum of all written values.
    """

    MIN_CAPACITY = 8

    def __init__(self, capacity: int, device: int | None = None) -> None:
        torch = _torch()
        cap = self.MIN_CAPACITY
        while cap < capacity:
            cap <<= 1
        self.capacity = cap
        self.device = torch.cuda.current_device() if device is None else int(device)
        self._kbuf = alloc(8 * cap, self.device)
        self._vbuf = alloc(8 * cap, self.device)
        self.keys = self._kbuf.tensor[: 8 * cap].view(torch.int64)
        self.vals = self._vbuf.tensor[: 8 * cap].view(torch.int64)
        self.keys.fill_(-1)  # NIL
        self.vals.zero_()
        self.count = 0
        self.peak_load = 0.0
        self._lib = _lib.load()

    def release(self) -> None:
        if self._kbuf is not None:
            release(self._kbuf)
            release(self._vbuf)
            self._kbuf = self._vbuf = None

    def grow(self, capacity: int) -> None:
        """Resize between rounds; only legal while empty."""
        if self.count:
            raise RuntimeError("reservation table can only grow while empty")
        if capacity <= self.capacity:
            return
        self.release()
        self.__init__(capacity, self.device)

    def _home(self, keys: np.ndarray) -> np.ndarray:
        shift = WORD(64 - self.capacity.bit_length() + 1)
        with np.errstate(over="ignore"):
            return (keys.astype(WORD) * WORD(GOLDEN)) >> shift

    def _note_load(self) -> None:
        load = self.count / self.capacity
        if load > self.peak_load:
            self.peak_load = load
        if 2 * self.count > self.capacity:
            raise RuntimeError("reservation table overfull; presize the table")

    def _stream(self) -> int:
        return _torch().cuda.current_stream(self.device).cuda_stream

    def reserve_max(self, keys, values, values_max_first: bool = False) -> None:
        """Per key, set the slot value to the max of the existing and the
        written values.  ``values_max_first`` is accepted for signature
        compatibility (the device algorithm needs no dedupe order)."""
        torch = _torch()
        if len(keys) != len(values):
            raise ValueError("keys/values length mismatch")
        if len(keys) == 0:
            return
        k, _ = _device_words(keys, self.device)
        v, _ = _device_words(values, self.device)
        n = k.numel()
        wb = self._lib.pip_rt_workspace_bytes(n)
        ws = torch.empty(wb, dtype=torch.uint8, device=f"cuda:{self.device}")
        cnt = C.c_uint64(0)
        with torch.cuda.device(self.device):
            rc = self._lib.pip_rt_reserve_max_u64(self.keys.data_ptr(), self.vals.data_ptr(),
                                                  self.capacity, k.data_ptr(), v.data_ptr(), n,
                                                  ws.data_ptr(), wb, C.byref(cnt), self._stream())
        if rc == _lib.PIP_ERR_TABLE:
            raise RuntimeError("reservation table probe overflow")
        _lib.check(rc, "reserve_max")
        self.count = int(cnt.value)
        self._note_load()

    def lookup(self, keys):
        """Return (values, found) for a batch of keys; absent keys get NIL.
        numpy in -> numpy out; CUDA tensor in -> CUDA tensors out."""
        torch = _torch()
        k, was_np = _device_words(keys, self.device)
        n = k.numel()
        out = torch.full((n,), -1, dtype=torch.int64, device=f"cuda:{self.device}")
        found = torch.zeros(n, dtype=torch.bool, device=f"cuda:{self.device}")
        if n and self.count:
            with torch.cuda.device(self.device):
                _lib.check(self._lib.pip_rt_lookup_u64(self.keys.data_ptr(), self.vals.data_ptr(),
                                                       self.capacity, k.data_ptr(), n, out.data_ptr(),
                                                       found.data_ptr(), self._stream()), "lookup")
        if was_np:
            return out.cpu().numpy().view(WORD), found.cpu().numpy()
        return out, found

    def delete(self, keys) -> None:
        """Clear the given keys' slots (part of a cleaning phase that removes
        every key inserted since the last clear, detres.py:165-193)."""
        torch = _torch()
        if len(keys) == 0 or self.count == 0:
            return
        k, _ = _device_words(keys, self.device)
        n = k.numel()
        wb = self._lib.pip_rt_workspace_bytes(n)
        ws = torch.empty(wb, dtype=torch.uint8, device=f"cuda:{self.device}")
        cnt = C.c_uint64(0)
        with torch.cuda.device(self.device):
            _lib.check(self._lib.pip_rt_delete_u64(self.keys.data_ptr(), self.capacity, k.data_ptr(),
                                                   n, ws.data_ptr(), wb, C.byref(cnt),
                                                   self._stream()), "delete")
        self.count = int(cnt.value)

    def clear(self) -> None:
        self.keys.fill_(-1)
        self.count = 0

    # scalar conveniences
    def put_max(self, key: int, value: int) -> None:
        self.reserve_max(np.array([key], dtype=WORD), np.array([value], dtype=WORD))

    def get(self, key: int) -> int | None:
        vals, found = self.lookup(np.array([key], dtype=WORD))
        return int(vals[0]) if found[0] else None

    def slot_keys(self) -> np.ndarray:
        """The key array as host words (NIL = empty): the slot layout."""
        return self.keys.cpu().numpy().view(WORD)


def reserve_max(table: ReservationTable, key: int, value: int) -> None:
    """Write-max a single key (linearizable per key)."""
    table.put_max(key, value)


# ---------------------------------------------------------------------------
# Round engine

@dataclass
class RoundStats:
    rounds: int = 0
    committed_per_round: list[int] = field(default_factory=list)
    peak_table_load: float = 0.0

    @property
    def total_committed(self) -> int:
        return sum(self.committed_per_round)


@dataclass
class RoundView:
    """State handed to the phase callbacks for one round (detres.py:233-240):
    ``ids`` (int64) and ``committed`` (bool) are CUDA tensor views of the
    engine's device buffers."""

    ids: object
    committed: object
    new_pos0: int
    round_index: int


def arange_source(n: int, device: int | None = None):
    """Default iterate source: ids 0..n-1 in ascending order, made on the device."""
    torch = _torch()
    dev = torch.cuda.current_device() if device is None else device
    state = {"next": 0}

    def source(count: int):
        lo = state["next"]
        hi = min(lo + count, n)
        state["next"] = hi
        return torch.arange(lo, hi, dtype=torch.int64, device=f"cuda:{dev}")

    return source


def run_rounds(n_iterates: int, prefix_size: int, reserve, commit, clean,
               id_source=None, trace: list | None = None, device: int | None = None) -> RoundStats:
    """Drive reserve/commit/clean rounds until all iterates are retired
    (detres.py:256-307).

    ``reserve``/``clean`` receive a :class:`RoundView`; ``commit`` must fill
    ``view.committed``.  Failures are packed in order on the device and the
    prefix is refilled from ``id_source`` (default: ascending ids; a source
    may return numpy words or CUDA tensors).  ``trace`` receives the committed
    ids of every round in packed order (CUDA tensors).
    """
    torch = _torch()
    if prefix_size < 1:
        raise ValueError("prefix size must be >= 1")
    dev = torch.cuda.current_device() if device is None else int(device)
    source = id_source if id_source is not None else arange_source(n_iterates, dev)
    prefix = max(1, min(prefix_size, n_iterates)) if n_iterates else 1
    lib = _lib.load()

    ids_buf = alloc(8 * prefix, dev)          # the reference's alloc(prefix)
    com_buf = alloc(prefix, dev)              # ... and alloc_bool(prefix)
    ids = ids_buf.tensor[: 8 * prefix].view(torch.int64)
    committed = com_buf.tensor[:prefix].view(torch.bool)
    tmp = torch.empty(prefix, dtype=torch.int64, device=f"cuda:{dev}") if trace is not None else None
    mdev = small_device_words(1, dev)
    stats = RoundStats()
    try:
        with torch.cuda.device(dev):
            st = torch.cuda.current_stream(dev).cuda_stream
            sp, sb = scratch_for(dev, st)
            fill = 0
            zero_rounds = 0
            while True:
                fresh = source(prefix - fill)
                new_pos0 = fill
                if len(fresh):
                    f, _ = _device_words(fresh, dev)
                    ids[fill:fill + f.numel()] = f
                    fill += f.numel()
                if fill == 0:
                    break
                view = RoundView(ids=ids[:fill], committed=committed[:fill], new_pos0=new_pos0,
                                 round_index=stats.rounds)
                view.committed.zero_()
                reserve(view)
                commit(view)
                clean(view)
                if trace is not None:
                    tmp[:fill] = ids[:fill]
                    _lib.check(lib.pip_compact_by_mask_u64(tmp.data_ptr(), fill,
                                                           committed.data_ptr(), mdev.data_ptr(),
                                                           sp, sb, st), "trace")
                    _lib.check_stall(sp, st, "trace")
                    trace.append(tmp[: int(mdev.item())].clone())
                keep = torch.logical_not(committed[:fill])
                _lib.check(lib.pip_compact_by_mask_u64(ids.data_ptr(), fill, keep.data_ptr(),
                                                       mdev.data_ptr(), sp, sb, st), "pack")
                _lib.check_stall(sp, st, "pack")
                left = int(mdev.item())
                ncommit = fill - left
                stats.rounds += 1
                stats.committed_per_round.append(ncommit)
                if ncommit == 0:
                    zero_rounds += 1
                    if zero_rounds >= LIVELOCK_ROUNDS:
                        raise LivelockError(
                            f"no iterate committed for {LIVELOCK_ROUNDS} rounds ({fill} active); "
                            "the client's commit rule cannot make progress")
                else:
                    zero_rounds = 0
                    fill = left
    finally:
        release(com_buf)
        release(ids_buf)
    return stats

