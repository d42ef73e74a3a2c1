"""Python face of the C oracle (oracle/pip_oracle.c).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, never by the product package.

Each function names the reference code it restates:
  seq_scan           baselines.py:26-35 (+ strong.py:132-166 generic op)
  seq_filter         baselines.py:38-41
  seq_knuth_shuffle  baselines.py:44-54
  seq_merge          baselines.py:99-114
  ref_scan           strong.py:107-166  (Alg. 3 up/down sweep, OpenMP tasks)
  ref_filter_kway    strong.py:283-349  (sqrt(n) chunks, batched moves)
  ref_merge_strong   strong.py:462-522  (split point + rotation recursion)
  ref_rotate         strong.py:67-95
  ref_random_permutation relaxed.py:64-251 + detres.py:256-307 (DR rounds)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "pip_oracle.c"
LIB = HERE / "_build" / "libpiporacle.so"

u64, u32, i32, vp = C.c_uint64, C.c_uint32, C.c_int, C.c_void_p
_lib = None

_SIGS = {
    "oracle_seq_scan": (None, [vp, vp, u64, i32, u64, i32, C.POINTER(u64)]),
    "oracle_seq_filter": (u64, [vp, u64, u32, u32, u64, u64, vp]),
    "oracle_seq_knuth_shuffle": (None, [vp, vp, u64]),
    "oracle_seq_merge": (None, [vp, u64, vp, u64, vp]),
    "oracle_ref_scan": (u64, [vp, u64, i32]),
    "oracle_ref_filter_kway": (u64, [vp, u64, u32, u32, u64, u64, i32]),
    "oracle_ref_partition_unstable": (u64, [vp, u64, u32, u32, u64, u64]),
    "oracle_ref_rotate": (None, [vp, u64, u64]),
    "oracle_ref_merge_strong": (None, [vp, u64, u64, i32]),
    "oracle_ref_random_permutation": (
        i32, [vp, vp, u64, u64, i32, vp, u64, vp, C.POINTER(u64), C.POINTER(u64),
              C.POINTER(u64), i32]),
    "oracle_max_threads": (i32, []),
}


def build(force: bool = False) -> Path:
    if LIB.exists() and not force and LIB.stat().st_mtime >= SRC.stat().st_mtime:
        return LIB
    LIB.parent.mkdir(parents=True, exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = ["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC", "-o", str(tmp),
           str(SRC)]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        lib = C.CDLL(str(LIB))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _w(a: np.ndarray) -> np.ndarray:
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a


OPS = {None: 0, "add": 0, "max": 1, "min": 2, "xor": 3}


def seq_scan(a: np.ndarray, op=None, init: int = 0, inclusive: bool = False):
    """Returns (out, total); ``a`` untouched."""
    a = _w(np.ascontiguousarray(a, dtype=np.uint64))
    out = np.empty_like(a)
    tot = u64(0)
    load().oracle_seq_scan(a.ctypes.data, out.ctypes.data, len(a), OPS[op], init & (2**64 - 1),
                           int(inclusive), C.byref(tot))
    return out, int(tot.value)


def seq_filter(a: np.ndarray, pred) -> np.ndarray:
    a = _w(np.ascontiguousarray(a, dtype=np.uint64))
    out = np.empty_like(a)
    m = load().oracle_seq_filter(a.ctypes.data, len(a), pred.kind, int(pred.negate), pred.a,
                                 pred.b, out.ctypes.data)
    return out[:m].copy()


def seq_knuth_shuffle(a: np.ndarray, h: np.ndarray) -> None:
    load().oracle_seq_knuth_shuffle(_w(a).ctypes.data, _w(h).ctypes.data, len(a))


def seq_merge(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    x = _w(np.ascontiguousarray(x, dtype=np.uint64))
    y = _w(np.ascontiguousarray(y, dtype=np.uint64))
    out = np.empty(len(x) + len(y), dtype=np.uint64)
    load().oracle_seq_merge(x.ctypes.data, len(x), y.ctypes.data, len(y), out.ctypes.data)
    return out


def ref_scan(a: np.ndarray, threads: int = 1) -> int:
    return int(load().oracle_ref_scan(_w(a).ctypes.data, len(a), threads))


def ref_filter_kway(a: np.ndarray, pred, threads: int = 1) -> int:
    return int(load().oracle_ref_filter_kway(_w(a).ctypes.data, len(a), pred.kind,
                                             int(pred.negate), pred.a, pred.b, threads))


def ref_partition_unstable(a: np.ndarray, pred) -> int:
    """strong.partition_unstable (strong.py:352-419), same output order."""
    return int(load().oracle_ref_partition_unstable(_w(a).ctypes.data, len(a), pred.kind,
                                                    int(pred.negate), pred.a, pred.b))


def ref_rotate(a: np.ndarray, o: int) -> None:
    load().oracle_ref_rotate(_w(a).ctypes.data, len(a), o)


def ref_merge_strong(a: np.ndarray, split: int, threads: int = 1) -> None:
    load().oracle_ref_merge_strong(_w(a).ctypes.data, len(a), split, threads)


VARIANTS = {"naive": 0, "flat": 1, "oneres": 2, "final": 3}


def ref_random_permutation(a: np.ndarray, h: np.ndarray, prefix: int, variant: str = "final",
                           threads: int = 1, want_trace: bool = False):
    """Returns dict(rounds, committed_per_round, peak_count, capacity, trace)."""
    n = len(a)
    counts = np.zeros(max(n, 1), dtype=np.uint64)
    trace = np.zeros(max(n, 1), dtype=np.uint64) if want_trace else None
    rounds, peak, cap = u64(0), u64(0), u64(0)
    rc = load().oracle_ref_random_permutation(
        _w(a).ctypes.data, _w(h).ctypes.data, n, prefix, VARIANTS[variant], counts.ctypes.data,
        len(counts), trace.ctypes.data if trace is not None else None, C.byref(rounds),
        C.byref(peak), C.byref(cap), threads)
    if rc == 2:
        raise ValueError("invalid swap sequence: H[i] must lie in [0, i]")
    if rc:
        raise RuntimeError(f"oracle rp failed with status {rc}")
    r = int(rounds.value)
    cpr = [int(x) for x in counts[:r]]
    out = {"rounds": r, "committed_per_round": cpr, "peak_count": int(peak.value),
           "capacity": int(cap.value)}
    if want_trace:
        tr, pos = [], 0
        for c in cpr:
            tr.append(trace[pos:pos + c].copy())
            pos += c
        out["trace"] = tr
    return out


def max_threads() -> int:
    return int(load().oracle_max_threads())
