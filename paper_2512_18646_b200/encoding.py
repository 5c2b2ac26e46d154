"""Layout types the column-ciphertext path returns (encoding.py:39-73 of the reference)."""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import EngineError


class Encoding(str, Enum):
    DATABASE = "database"
    ROW_MAJOR = "row-major"
    REVOLVER = "revolver"


@dataclass(frozen=True)
class MatrixShape:
    m: int
    n: int

    def __post_init__(self):
        if self.m < 1 or self.n < 1:
            raise EngineError(f"matrix shape must be positive, got {self.m}x{self.n}")


@dataclass(frozen=True, eq=False)
class PackedMatrix:
    """A ciphertext holding an m x n matrix in its leading m*n slots."""

    ct: object
    shape: MatrixShape
    encoding: Encoding
    revolve_p: int | None = None

    def decode(self, engine) -> np.ndarray:
        m, n = self.shape.m, self.shape.n
        return engine.dec(self.ct)[: m * n].reshape(m, n)

    def with_ct(self, ct) -> "PackedMatrix":
        return PackedMatrix(ct, self.shape, self.encoding, self.revolve_p)


@dataclass(frozen=True, eq=False)
class Kernel:
    """Dense square kernel plus bias (conv.py:46-61 of the reference)."""

    weights: np.ndarray
    bias: float = 0.0

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=np.float64)
        if w.ndim != 2 or w.shape[0] != w.shape[1] or w.shape[0] < 1:
            raise EngineError(f"kernel must be square, got shape {w.shape}")
        object.__setattr__(self, "weights", w)

    @property
    def k(self) -> int:
        return self.weights.shape[0]
