"""Round statistics and errors of the deterministic-reservations engine.

Mirrors ``pipal.detres`` (reference detres.py:30-34, :222-240).  The engine
itself (reserve / commit / clean / pack rounds, detres.py:256-307) runs on the
GPU inside ``libpip`` (csrc/rp.cu) as one persistent cooperative kernel; these
are the host-side result types it reports through.
"""
from __future__ import annotations

from dataclasses import dataclass, field

LIVELOCK_ROUNDS = 64

__all__ = ["RoundStats", "LivelockError", "LIVELOCK_ROUNDS"]


class LivelockError(RuntimeError):
    """No iterate committed for LIVELOCK_ROUNDS consecutive rounds."""


@dataclass
class RoundStats:
    rounds: int = 0
    committed_per_round: list[int] = field(default_factory=list)
    peak_table_load: float = 0.0

    @property
    def total_committed(self) -> int:
        return sum(self.committed_per_round)
