"""Runtime support mirroring ``pipal.runtime`` (reference runtime.py).

Kept from the reference, with the same names and semantics:
  * word validation (``as_words`` — runtime.py:45-51): numpy arrays must be
    1-D C-contiguous uint64; additionally torch CUDA tensors (uint64 or int64,
    1-D, contiguous) are accepted and processed in place on the device;
  * the auxiliary-space meter (``SpaceMeter``, ``meter_scope``, ``metered``,
    ``alloc``/``release``/``aux`` — runtime.py:164-253), charging
    ceil(bytes / 8) words per buffer; here the buffers are DEVICE workspace;
  * the counter-based RNG (``Rng`` — runtime.py:263-302), bit-identical on
    host (numpy) and device (``Rng.words_device``);
  * ``EpsilonConfig`` budgets b(n) (runtime.py:311-329).
The fork-join pool (runtime.py:60-158) has no GPU counterpart: results are
independent of it, ``set_num_threads`` is accepted and recorded only.
"""
from __future__ import annotations

import math
import threading
from contextlib import contextmanager
from dataclasses import dataclass

import numpy as np

from . import _lib

WORD = np.uint64
M64 = (1 << 64) - 1
NIL = M64
GOLDEN = 0x9E3779B97F4A7C15
SCRATCH_WORDS = 256

__all__ = [
    "WORD", "M64", "NIL", "SCRATCH_WORDS", "GOLDEN",
    "as_words", "make_words", "Words",
    "set_num_threads", "num_threads",
    "SpaceMeter", "MeterReport", "meter_scope", "metered", "alloc", "release", "aux",
    "Rng", "EpsilonConfig", "POWER_ONLY_FRACTION", "compact_by_mask",
]


# ---------------------------------------------------------------------------
# word arrays: numpy (host, reference-compatible) or torch CUDA (device)

def _torch():
    import torch

    return torch


class Words:
    """A validated word array: host numpy buffer or device torch tensor."""

    __slots__ = ("obj", "n", "ptr", "device", "is_device")

    def __init__(self, obj, n, ptr, device, is_device):
        self.obj = obj
        self.n = n
        self.ptr = ptr
        self.device = device
        self.is_device = is_device

    def stream(self):
        torch = _torch()
        return torch.cuda.current_stream(self.device).cuda_stream

    def to_numpy(self) -> np.ndarray:
        if not self.is_device:
            return self.obj
        t = self.obj
        torch = _torch()
        if t.dtype == torch.uint64:
            t = t.view(torch.int64)
        return t.cpu().numpy().view(np.uint64)


def _is_torch_tensor(a) -> bool:
    try:
        torch = _torch()
    except Exception:  # pragma: no cover
        return False
    return isinstance(a, torch.Tensor)


def as_words(a, _wrap: bool = False):
    """Validate ``a`` as a mutable 1-D contiguous word array (runtime.py:45-51).

    numpy: must be uint64, 1-D, C-contiguous (TypeError otherwise, as in the
    reference).  torch: must be a CUDA tensor of uint64 or int64, 1-D,
    contiguous (int64 buffers are reinterpreted as unsigned words).
    """
    if isinstance(a, np.ndarray):
        if a.dtype != WORD or a.ndim != 1:
            raise TypeError("expected a 1-D numpy array of uint64 words")
        if not a.flags.c_contiguous:
            raise TypeError("word arrays must be C-contiguous")
        if not a.flags.writeable:
            raise TypeError("word arrays must be writeable")
        return Words(a, len(a), a.ctypes.data, None, False) if _wrap else a
    if _is_torch_tensor(a):
        torch = _torch()
        if a.dtype not in (torch.uint64, torch.int64) or a.dim() != 1:
            raise TypeError("expected a 1-D torch tensor of uint64/int64 words")
        if not a.is_cuda:
            raise TypeError("torch word tensors must live on a CUDA device")
        if not a.is_contiguous():
            raise TypeError("word arrays must be contiguous")
        return Words(a, a.numel(), a.data_ptr(), a.device.index, True) if _wrap else a
    raise TypeError("expected a 1-D numpy array of uint64 words")


def make_words(values) -> np.ndarray:
    return np.array([int(v) & M64 for v in values], dtype=WORD)


# ---------------------------------------------------------------------------
# thread-count knob (reference fork-join pool): recorded only

_threads = 1


def set_num_threads(n: int) -> None:
    global _threads
    if n < 1:
        raise ValueError("thread count must be >= 1")
    _threads = n


def num_threads() -> int:
    return _threads


# ---------------------------------------------------------------------------
# space metering (runtime.py:164-253)

@dataclass
class MeterReport:
    peak_words: int
    budget_words: int
    exceeded: bool


class SpaceMeter:
    """Counts auxiliary heap words held by instrumented operations."""

    def __init__(self) -> None:
        self.current_words = 0
        self.peak_words = 0
        self._lock = threading.Lock()

    def acquire(self, words: int) -> None:
        if words < 0:
            raise ValueError("cannot acquire a negative word count")
        with self._lock:
            self.current_words += words
            if self.current_words > self.peak_words:
                self.peak_words = self.current_words

    def release(self, words: int) -> None:
        with self._lock:
            self.current_words -= words
            if self.current_words < 0:
                raise RuntimeError("space meter released more than acquired")


_meter_stack: list[SpaceMeter] = []


@contextmanager
def metered(meter: SpaceMeter):
    _meter_stack.append(meter)
    try:
        yield meter
    finally:
        _meter_stack.pop()


def _active_meter() -> SpaceMeter | None:
    return _meter_stack[-1] if _meter_stack else None


def meter_scope(meter: SpaceMeter, budget_words: int, body) -> MeterReport:
    """Run ``body`` with ``meter`` active; never aborts on budget overrun."""
    with metered(meter):
        body()
    return MeterReport(peak_words=meter.peak_words, budget_words=budget_words,
                       exceeded=meter.peak_words > budget_words)


def _charge_words(nbytes: int) -> int:
    return (nbytes + 7) // 8


def _caller_meter():
    """The reference's own active meter, when the caller runs inside
    ``pipal.runtime.metered`` / ``meter_scope`` (runtime.py:194-207): GPU
    workspace is charged to it too, so a pipal user measuring a drop-in call
    sees its words (not only users of this package's meter)."""
    import sys

    ref = sys.modules.get("pipal.runtime")
    stack = getattr(ref, "_meter_stack", None) if ref is not None else None
    return stack[-1] if stack else None


def _active_meters() -> list:
    out = []
    m = _active_meter()
    if m is not None:
        out.append(m)
    c = _caller_meter()
    if c is not None and all(c is not x for x in out):
        out.append(c)
    return out


class DeviceBuffer:
    """Charged device workspace (the GPU counterpart of runtime.alloc)."""

    __slots__ = ("tensor", "nbytes", "words", "_released", "_meters")

    def __init__(self, nbytes: int, device: int):
        torch = _torch()
        self.nbytes = int(nbytes)
        self.tensor = torch.empty(max(self.nbytes, 16), dtype=torch.uint8, device=f"cuda:{device}")
        self.words = _charge_words(self.nbytes)
        self._released = False
        self._meters = _active_meters()
        for m in self._meters:
            m.acquire(self.words)

    @property
    def ptr(self) -> int:
        return self.tensor.data_ptr()


def alloc(nbytes: int, device: int) -> DeviceBuffer:
    return DeviceBuffer(nbytes, device)


def charge(words: int) -> list:
    """Charge words for workspace allocated inside a host-path C call;
    returns the meters charged (pass them to ``uncharge``)."""
    ms = _active_meters()
    for m in ms:
        m.acquire(words)
    return ms


def uncharge(words: int, meters: list | None = None) -> None:
    for m in (meters if meters is not None else _active_meters()):
        m.release(words)


def release(buf: DeviceBuffer) -> None:
    if buf._released:
        return
    buf._released = True
    for m in buf._meters:
        m.release(buf.words)
    buf.tensor = None


@contextmanager
def aux(nbytes: int, device: int):
    buf = alloc(nbytes, device)
    try:
        yield buf
    finally:
        release(buf)


# ---------------------------------------------------------------------------
# unmetered O(#CTAs) scratch, one per (device, stream)

_scratch: dict[tuple[int, int], object] = {}


def scratch_for(device: int, stream: int):
    """(ptr, nbytes) of the strong ops' look-back scratch on this stream."""
    key = (device, stream)
    t = _scratch.get(key)
    lib = _lib.load()
    nbytes = lib.pip_scratch_bytes(device)
    if t is None:
        torch = _torch()
        t = torch.zeros(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
        _scratch[key] = t
    return t.data_ptr(), nbytes


def small_device_words(k: int, device: int):
    torch = _torch()
    return torch.zeros(k, dtype=torch.int64, device=f"cuda:{device}")


# ---------------------------------------------------------------------------
# counter-based RNG (runtime.py:263-302)

def _mix64_scalar(z: int) -> int:
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> WORD(30))
    z = z * WORD(0xBF58476D1CE4E5B9)
    z = z ^ (z >> WORD(27))
    z = z * WORD(0x94D049BB133111EB)
    return z ^ (z >> WORD(31))


class Rng:
    """Deterministic counter-based random words: value(seed, i) is pure."""

    __slots__ = ("seed",)

    def __init__(self, seed: int) -> None:
        self.seed = int(seed) & M64

    def word(self, i: int) -> int:
        return _mix64_scalar(self.seed + (i + 1) * GOLDEN)

    def words(self, lo: int, hi: int) -> np.ndarray:
        idx = np.arange(lo + 1, hi + 1, dtype=WORD)
        with np.errstate(over="ignore"):
            return _mix64((idx * WORD(GOLDEN)) + WORD(self.seed))

    def words_at(self, idx: np.ndarray) -> np.ndarray:
        with np.errstate(over="ignore"):
            z = (idx.astype(WORD) + WORD(1)) * WORD(GOLDEN) + WORD(self.seed)
            return _mix64(z)

    def below(self, i: int, bound: int) -> int:
        return self.word(i) % bound

    def derive(self, tag: int) -> "Rng":
        return Rng(_mix64_scalar(self.seed ^ _mix64_scalar(tag)))

    # device generation (same values as words(lo, hi) >> shift)
    def words_device(self, lo: int, hi: int, shift: int = 0, device: int = 0, out=None):
        torch = _torch()
        n = hi - lo
        t = out if out is not None else torch.empty(n, dtype=torch.int64, device=f"cuda:{device}")
        lib = _lib.load()
        st = torch.cuda.current_stream(t.device).cuda_stream
        _lib.check(lib.pip_rng_words_u64(t.data_ptr(), lo, n, self.seed, shift, st), "rng_words")
        return t

    def swaps_device(self, lo: int, hi: int, device: int = 0, out=None):
        """relaxed.make_swap_sequence on the device: H[i] = words[i] % (i+1)."""
        torch = _torch()
        n = hi - lo
        t = out if out is not None else torch.empty(n, dtype=torch.int64, device=f"cuda:{device}")
        lib = _lib.load()
        st = torch.cuda.current_stream(t.device).cuda_stream
        _lib.check(lib.pip_make_swaps_u64(t.data_ptr(), lo, n, self.seed, st), "make_swaps")
        return t


# ---------------------------------------------------------------------------
# relaxed-model budgets (runtime.py:311-329)

POWER_ONLY_FRACTION = 1e-12


@dataclass(frozen=True)
class EpsilonConfig:
    """Auxiliary-space budget b(n) = max(ceil(n^(1-epsilon)), floor(f*n))."""

    epsilon: float
    prefix_fraction: float = 0.02

    def __post_init__(self) -> None:
        if not 0.0 < self.epsilon < 1.0:
            raise ValueError("epsilon must lie in (0, 1)")
        if not 0.0 < self.prefix_fraction <= 1.0:
            raise ValueError("prefix_fraction must lie in (0, 1]")

    def prefix_words(self, n: int) -> int:
        if n < 1:
            return 1
        b = max(math.ceil(n ** (1.0 - self.epsilon)), math.floor(self.prefix_fraction * n))
        return min(max(b, 1), n)


# ---------------------------------------------------------------------------
# shared in-place primitive (runtime.py:335-355)

def compact_by_mask(arr, keep, n: int | None = None) -> int:
    """Stable in-place compaction of arr[i] with keep[i]; returns the new count.

    Runs on the device (``pip_compact_by_mask_u64``: the look-back filter
    with the keep flags read from a byte mask, O(#CTAs) scratch, zero heap
    like the reference's SCRATCH_WORDS blocks).  ``arr``: numpy uint64 (copied
    through the device and back in place) or a CUDA int64/uint64 tensor;
    ``keep``: a bool / uint8 array of at least ``n`` flags (numpy or CUDA).
    Only arr[0:n) is compacted; arr[m:n) is unspecified afterwards.
    """
    w: Words = as_words(arr, _wrap=True)
    n = w.n if n is None else int(n)
    if n < 0 or n > w.n or len(keep) < n:
        raise ValueError("n out of range")
    if n == 0:
        return 0
    torch = _torch()
    lib = _lib.load()
    if not w.is_device:
        dev = torch.cuda.current_device()
        t = torch.from_numpy(w.obj[:n].view(np.int64)).to(f"cuda:{dev}")
        m = compact_by_mask(t, keep, n)
        w.obj[:m] = t[:m].cpu().numpy().view(np.uint64)
        return m
    if isinstance(keep, np.ndarray):
        k = torch.from_numpy(np.ascontiguousarray(keep[:n]).view(np.uint8)).to(f"cuda:{w.device}")
    else:
        k = keep[:n]
        if k.device != w.obj.device:
            raise ValueError("keep mask must live on the array's device")
        k = (k.view(torch.uint8) if k.dtype == torch.bool else k.to(torch.uint8)).contiguous()
    with torch.cuda.device(w.device):
        st = w.stream()
        sp, sb = scratch_for(w.device, st)
        out = small_device_words(1, w.device)
        _lib.check(lib.pip_compact_by_mask_u64(w.ptr, n, k.data_ptr(), out.data_ptr(), sp, sb, st),
                   "compact_by_mask")
        _lib.check_stall(sp, st, "compact_by_mask")
        return int(out.item())
