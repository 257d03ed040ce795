"""``ScanProblem`` and ``ShapeError`` — mirror of chainscan/reference.py:34-58."""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from ._compat import compat


class ShapeError(ValueError):
    """Raised when an input shape violates a precondition (reference.py:34-35)."""


@dataclass
class ScanProblem:
    """An inclusive-scan instance: 1-D input x, operator op, optional out.

    When out is given the result is written there (it may alias x for an
    in-place scan); otherwise a fresh array is allocated (reference.py:38-58).
    """

    x: np.ndarray
    op: object
    out: Optional[np.ndarray] = None

    def __post_init__(self):
        self.x = np.asanyarray(self.x)
        if self.x.ndim != 1:
            raise compat(ShapeError)(f"input must be 1-D, got shape {self.x.shape}")
        if self.out is not None and self.out.shape != self.x.shape:
            raise compat(ShapeError)("out shape must match input shape")

    def resolve_out(self) -> np.ndarray:
        return self.out if self.out is not None else np.empty_like(self.x)
