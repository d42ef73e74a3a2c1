"""B200-native parallel in-place (PIP) kernels — drop-in for the hot path of
``pipal`` (arXiv 2103.01216 reference): random permutation by deterministic
reservations, in-place scan, stable in-place filter, in-place merge; plus
unstable partition / quicksort and list contraction / ranking on the same
engines.

Compute runs in hand-written sm_100a CUDA behind a C ABI (include/pip.h,
libpip.so); this package mirrors the reference's module layout and function
signatures: ``strong``, ``relaxed``, ``detres``, ``runtime``, ``contraction``, plus the
``.u64`` container / report CSV (``formats``) and the command-line harness
(``python -m paper_2103_01216_b200.cli``).
"""
from . import _lib, detres, formats, pred, runtime, strong, relaxed  # noqa: F401
from . import contraction  # noqa: F401
from .detres import LivelockError, RoundStats
from .pred import Pred
from .runtime import EpsilonConfig, MeterReport, Rng, SpaceMeter, as_words, meter_scope

__all__ = ["strong", "relaxed", "detres", "runtime", "contraction", "pred", "formats", "Pred", "EpsilonConfig", "Rng",
           "SpaceMeter", "MeterReport", "meter_scope", "as_words", "RoundStats", "LivelockError"]
