"""Predicate descriptors for the filter kernels.

The reference passes arbitrary numpy callables (``cli.py:41`` EVEN,
``test_strong.py:21,184``, ``strong.py:440-441,553``).  A GPU kernel cannot
run a Python callable, and there is no CPU fallback, so the drop-in takes a
``Pred``: a small descriptor that the kernel evaluates
(``pip_pred`` in include/pip.h) and that is ALSO a numpy callable with the
reference's calling convention ``pred(block) -> bool mask``, so the same
object drives the reference/oracle in tests.  Plain callables raise
``TypeError``.
"""
from __future__ import annotations

import numpy as np

from . import _lib

WORD = np.uint64
M64 = (1 << 64) - 1


class Pred:
    __slots__ = ("kind", "a", "b", "negate", "name")

    def __init__(self, kind: int, a: int = 0, b: int = 0, negate: bool = False, name: str = ""):
        self.kind = int(kind)
        self.a = int(a) & M64
        self.b = int(b) & M64
        self.negate = bool(negate)
        self.name = name or f"pred{kind}"

    # numpy semantics (identical results to the kernel)
    def __call__(self, block: np.ndarray) -> np.ndarray:
        x = np.asarray(block, dtype=WORD)
        a, b = WORD(self.a), WORD(self.b)
        k = self.kind
        if k == _lib.PRED_ALL:
            r = np.ones(x.shape, dtype=bool)
        elif k == _lib.PRED_MASK_EQ:
            r = (x & a) == b
        elif k == _lib.PRED_MOD_EQ:
            r = (x % a) == b
        elif k == _lib.PRED_LT:
            r = x < a
        elif k == _lib.PRED_LE:
            r = x <= a
        elif k == _lib.PRED_GT:
            r = x > a
        elif k == _lib.PRED_GE:
            r = x >= a
        elif k == _lib.PRED_EQ:
            r = x == a
        else:  # pragma: no cover
            raise ValueError(f"unknown predicate kind {k}")
        return ~r if self.negate else r

    def __invert__(self) -> "Pred":
        return Pred(self.kind, self.a, self.b, not self.negate, f"~{self.name}")

    def descriptor(self) -> _lib.PipPred:
        return _lib.PipPred(self.kind, 1 if self.negate else 0, self.a, self.b)

    def __repr__(self) -> str:
        return f"Pred({self.name})"


def as_pred(pred) -> Pred:
    if isinstance(pred, Pred):
        return pred
    raise TypeError(
        "GPU filters need a Pred descriptor (even(), odd(), mod_eq(k, r), lt(v), le(v), "
        "gt(v), ge(v), eq(v), bit_set(b), bit_clear(b), mask_eq(m, v), always()); "
        "arbitrary Python callables cannot run on the device and there is no CPU fallback")


def even() -> Pred:
    """cli.py:41 EVEN: (b & 1) == 0"""
    return Pred(_lib.PRED_MASK_EQ, 1, 0, name="even")


def odd() -> Pred:
    """test_strong.py:184: (b & 1) == 1"""
    return Pred(_lib.PRED_MASK_EQ, 1, 1, name="odd")


def mask_eq(mask: int, value: int) -> Pred:
    return Pred(_lib.PRED_MASK_EQ, mask, value, name=f"mask_eq({mask:#x},{value:#x})")


def bit_set(bit: int) -> Pred:
    return Pred(_lib.PRED_MASK_EQ, 1 << bit, 1 << bit, name=f"bit_set({bit})")


def bit_clear(bit: int) -> Pred:
    return Pred(_lib.PRED_MASK_EQ, 1 << bit, 0, name=f"bit_clear({bit})")


def mod_eq(k: int, r: int) -> Pred:
    """x % k == r  (BASELINE config 2 keeps x % 3 == 0)"""
    if k < 1:
        raise ValueError("modulus must be >= 1")
    return Pred(_lib.PRED_MOD_EQ, k, r, name=f"mod_eq({k},{r})")


def lt(v: int) -> Pred:
    """strong.py:440: b < pivot"""
    return Pred(_lib.PRED_LT, v, name=f"lt({v})")


def le(v: int) -> Pred:
    return Pred(_lib.PRED_LE, v, name=f"le({v})")


def gt(v: int) -> Pred:
    return Pred(_lib.PRED_GT, v, name=f"gt({v})")


def ge(v: int) -> Pred:
    return Pred(_lib.PRED_GE, v, name=f"ge({v})")


def eq(v: int) -> Pred:
    """strong.py:441: b == pivot"""
    return Pred(_lib.PRED_EQ, v, name=f"eq({v})")


def always() -> Pred:
    return Pred(_lib.PRED_ALL, name="always")


EVEN = even()
ODD = odd()
