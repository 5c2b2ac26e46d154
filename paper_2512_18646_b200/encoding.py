"""Layout types the column-ciphertext path returns (encoding.py:39-73 of the reference)."""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import CapacityError, EngineError


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

    def decode_async(self, engine):
        """``decode`` as a future (CkksEngine.dec_batch_async): ``.result()`` returns the matrix."""
        m, n = self.shape.m, self.shape.n
        return engine.dec_batch_async([self.ct], post=lambda v: v[0][: m * n].reshape(m, n).copy())

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


# ---- row-major / revolver packing and the rotate-and-add primitives (encoding.py:90-170) ----
# Written against the SlotEngine surface (enc/rot/add/cmul/mask) plus CkksEngine's batched forms
# (rot_batch/add_batch/cmul_batch): one launch per cascade step for all matrices.

def _fits(engine, m: int, n: int) -> None:
    if m * n > engine.slots:
        raise CapacityError(f"{m}x{n} matrix needs {m * n} slots, engine has {engine.slots}")


def _as_matrix(x) -> np.ndarray:
    return np.atleast_2d(np.asarray(x, dtype=np.float64))


def encode_db(engine, z) -> PackedMatrix:
    """Database layout: the matrix row by row in the leading slots (encoding.py:81-87)."""
    z = _as_matrix(z)
    m, n = z.shape
    _fits(engine, m, n)
    return PackedMatrix(engine.enc(z.reshape(-1), layout=("grid", m, n)), MatrixShape(m, n), Encoding.DATABASE)


def encode_row_major(engine, a) -> PackedMatrix:
    """Left matmul operand: plain row-major packing (encoding.py:90-96)."""
    a = _as_matrix(a)
    m, n = a.shape
    _fits(engine, m, n)
    return PackedMatrix(engine.enc(a.reshape(-1), layout=("grid", m, n)), MatrixShape(m, n), Encoding.ROW_MAJOR)


def encode_revolver(engine, b, target_m: int) -> PackedMatrix:
    """Right operand in the revolver layout: layout row r = column (r mod p) of B (encoding.py:99-118)."""
    b = _as_matrix(b)
    n, p = b.shape
    if target_m < 1:
        raise EngineError("target_m must be positive")
    _fits(engine, target_m, n)
    grid = b.T[np.arange(target_m) % p]
    return PackedMatrix(engine.enc(grid.reshape(-1), layout=("grid", target_m, n)), MatrixShape(target_m, n),
                        Encoding.REVOLVER, revolve_p=p)


def incomplete_col_shift(engine, pm: PackedMatrix) -> PackedMatrix:
    """Packed entry stream moved left by one slot (encoding.py:121-129)."""
    return pm.with_ct(engine.rot(pm.ct, 1))


def row_shift(engine, pm: PackedMatrix) -> PackedMatrix:
    """Every row up by one position: rotation by the row width (encoding.py:132-134)."""
    return pm.with_ct(engine.rot(pm.ct, pm.shape.n))


def _log2_exact(x: int, what: str) -> int:
    if x < 1 or x & (x - 1):
        raise EngineError(f"{what} requires a power-of-two {'row' if what == 'sum_row_vec' else 'column'} count, got {x}")
    return x.bit_length() - 1


def sum_row_vec(engine, pm: PackedMatrix) -> PackedMatrix:
    """Column sums replicated into every row: log2(m) rotate-and-add steps (encoding.py:137-151)."""
    m, n = pm.shape.m, pm.shape.n
    ct = pm.ct
    for t in range(_log2_exact(m, "sum_row_vec")):
        ct = engine.add(ct, engine.rot(ct, n << t))
    return pm.with_ct(ct)


def _col0_filter(engine, m: int, n: int):
    grid = np.zeros((m, n))
    grid[:, 0] = 1.0
    return engine.mask(grid.reshape(-1), role="filter")


def sum_col_vec(engine, pm: PackedMatrix) -> PackedMatrix:
    """Each row replaced by its sum (encoding.py:154-170): a rotate-and-add cascade collects the
    row sum in column 0, a 0/1 filter keeps column 0, and a reverse cascade spreads it back.
    2*log2(n) rotations, 2*log2(n) adds, one cmul."""
    return sum_col_vec_many(engine, [pm])[0]


def sum_col_vec_many(engine, pms) -> list[PackedMatrix]:
    """sum_col_vec of several same-shape matrices; one batched launch per cascade step on the GPU."""
    pms = list(pms)
    if not pms:
        return []
    m, n = pms[0].shape.m, pms[0].shape.n
    steps = _log2_exact(n, "sum_col_vec")
    cts = [pm.ct for pm in pms]
    for t in range(steps):
        cts = engine.add_batch(cts, [r[0] for r in engine.rot_batch(cts, [1 << t])])
    keep = _col0_filter(engine, m, n)
    cts = engine.cmul_batch(keep, cts)
    for t in range(steps):
        cts = engine.add_batch(cts, [r[0] for r in engine.rot_batch(cts, [-(1 << t)])])
    return [pm.with_ct(c) for pm, c in zip(pms, cts)]


def matrix_from_csv(path) -> np.ndarray:
    """Dense matrix from CSV, one row per line (encoding.py:173-175)."""
    return np.loadtxt(path, delimiter=",", dtype=np.float64, ndmin=2)
