"""Migration plan types (reference: migration.py:35-75).  The planner and the
executor that consumes these plans are in planner.py / reshard.py."""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction


class MigrationError(ValueError):
    """(reference: migration.py:35-36)"""


@dataclass(frozen=True)
class Transfer:
    """(reference: migration.py:39-51)"""

    kind: str
    layer: int
    lo: Fraction
    hi: Fraction
    src: tuple
    dst: tuple
    bytes: float
    request: str | None = None
    tokens: int = 0


@dataclass(frozen=True)
class MigrationAction:
    """(reference: migration.py:54-62)"""

    kind: str
    transfers: tuple = ()
    releases: tuple = ()
    layer: int | None = None
    stage: int | None = None


@dataclass
class MigrationPlan:
    """(reference: migration.py:65-75)"""

    actions: list
    u_max: float | None = None
    peak_usage: dict = field(default_factory=dict)

    def transfers(self) -> list:
        return [t for a in self.actions for t in a.transfers]

    def total_bytes(self) -> float:
        return sum(t.bytes for t in self.transfers())
