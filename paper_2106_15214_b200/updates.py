"""Update-family enums and instrumentation of the reference ``betanmf.updates``.

The update kernels themselves live in libbnmf (csrc/); this module keeps the
host-visible names: ``Algorithm`` (updates.py:37-39), ``OpCounter``
(updates.py:42-57) and ``UpdateKind`` (updates.py:60-81).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

from .core import gamma_exponent


class Algorithm(str, Enum):
    BMM = "bmm"
    JMM = "jmm"


@dataclass
class OpCounter:
    """Counts products and kernel calls (updates.py:42-57).  The device runs
    a fixed schedule, so the counts are added per finished outer iteration
    exactly as the reference's kernels would increment them."""

    kernel_products: int = 0
    anchor_products: int = 0
    objective_products: int = 0
    w_updates: int = 0
    h_updates: int = 0

    def reset(self):
        self.kernel_products = 0
        self.anchor_products = 0
        self.objective_products = 0
        self.w_updates = 0
        self.h_updates = 0


@dataclass
class UpdateKind:
    """Which update family to run and how (updates.py:60-81)."""

    algorithm: Algorithm
    use_fast_path: bool | None = None
    heuristic_gamma_one: bool = False

    def fast_path_enabled(self, beta):
        if self.use_fast_path is None:
            return beta in (0.0, 1.0, 2.0)
        return self.use_fast_path

    def exponent(self, beta):
        return 1.0 if self.heuristic_gamma_one else gamma_exponent(beta)
