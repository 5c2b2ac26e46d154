"""Engine parameters: the reference's EngineParams (engine.py:54-90) extended
with the RNS-CKKS prime chain.

``slots``, ``log_q``, ``log_n``, ``delta`` and ``delta_c`` keep their reference
meaning (slots = N/2, log_n = log2(2*slots)); the chain defaults are derived
from them so ``EngineParams(slots=...)`` behaves like the reference factory
(tests/conftest.py:7-8).  Extra fields:

* ``prime_bits``   bit sizes of q0..qL (default: 60, then ``delta``-bit primes
                   filling ``log_q`` minus the q0 and special-prime budget)
* ``special_bits`` bit size of the key-switching prime P (default 60)
* ``seed``         seed of every key and encryption sample
* ``encryption``   "secret" (key-owner encryption, 1 NTT per limb, default) or "public" (pk)
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from pathlib import Path

from .errors import EngineError


def is_pow2(x: int) -> bool:
    return x > 0 and (x & (x - 1)) == 0


def next_pow2(x: int) -> int:
    if x <= 1:
        return 1
    return 1 << (x - 1).bit_length()


_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 2^64."""
    if n < 2:
        return False
    for p in _MR_BASES:
        if n % p == 0:
            return n == p
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in _MR_BASES:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def gen_primes(log_n: int, bits) -> list[int]:
    """For each bit size in order: largest prime < 2^bits, == 1 mod 2N, not yet taken."""
    two_n = 2 << log_n
    out: list[int] = []
    for b in bits:
        if b < log_n + 2 or b > 61:
            raise EngineError(f"prime size {b} unsupported for log_n={log_n} (need log_n+2 <= bits <= 61)")
        top = (1 << b) - 1
        c = (top // two_n) * two_n + 1
        if c > top:
            c -= two_n
        while True:
            if c < two_n:
                raise EngineError(f"ran out of {b}-bit NTT primes")
            if c not in out and is_prime(c):
                break
            c -= two_n
        out.append(c)
    return out


@dataclass(frozen=True)
class EngineParams:
    slots: int = 32768
    log_q: int = 1200
    log_n: int | None = None
    delta: int = 45
    delta_c: int = 20
    prime_bits: tuple | None = None
    special_bits: int = 60
    seed: int = 0
    encryption: str = "secret"
    primes: tuple = field(init=False, repr=False, compare=False, default=())

    def __post_init__(self):
        if not is_pow2(self.slots) or self.slots < 2:
            raise EngineError(f"slots must be a power of two >= 2, got {self.slots}")
        expect = int(math.log2(2 * self.slots))
        if self.log_n is None:
            object.__setattr__(self, "log_n", expect)
        elif self.log_n != expect:
            raise EngineError(f"log_n={self.log_n} must equal log2(2*slots)={expect} for CKKS")
        if self.encryption not in ("public", "secret"):
            raise EngineError(f"encryption must be 'public' or 'secret', got {self.encryption!r}")
        if self.prime_bits is None:
            levels = max(1, (self.log_q - 60 - self.special_bits) // self.delta)
            bits = (60,) + (self.delta,) * levels
            object.__setattr__(self, "prime_bits", bits)
        else:
            object.__setattr__(self, "prime_bits", tuple(int(b) for b in self.prime_bits))
        if len(self.prime_bits) < 1 or len(self.prime_bits) + 1 > 39:
            raise EngineError("prime chain must have 1..38 ciphertext primes")
        primes = gen_primes(self.log_n, list(self.prime_bits) + [self.special_bits])
        object.__setattr__(self, "primes", tuple(primes))

    @property
    def levels(self) -> int:
        """Top level L (ciphertext primes q0..qL)."""
        return len(self.prime_bits) - 1

    @property
    def n(self) -> int:
        return 2 * self.slots

    @property
    def scale(self) -> float:
        return float(2 ** self.delta)

    def scale_chain(self) -> list[float]:
        """Canonical scale per level: s[L] = 2^delta, s[l-1] = s[l]^2 / q[l]."""
        L = self.levels
        s = [0.0] * (L + 1)
        s[L] = self.scale
        for lv in range(L, 0, -1):
            s[lv - 1] = (s[lv] * s[lv]) / float(self.primes[lv])
        return s

    @classmethod
    def from_config(cls, path) -> "EngineParams":
        """JSON loader with the reference's keys (engine.py:76-90) plus chain keys."""
        raw = json.loads(Path(path).read_text())
        known = {"slots", "logq", "logn", "delta", "delta_c", "prime_bits", "special_bits", "seed", "encryption"}
        unknown = sorted(set(raw) - known)
        if unknown:
            raise EngineError(f"unknown config keys in {path}: {unknown}")
        return cls(
            slots=int(raw.get("slots", 32768)),
            log_q=int(raw.get("logq", 1200)),
            log_n=int(raw["logn"]) if "logn" in raw else None,
            delta=int(raw.get("delta", 45)),
            delta_c=int(raw.get("delta_c", 20)),
            prime_bits=tuple(raw["prime_bits"]) if "prime_bits" in raw else None,
            special_bits=int(raw.get("special_bits", 60)),
            seed=int(raw.get("seed", 0)),
            encryption=str(raw.get("encryption", "secret")),
        )


def config_params(cfg: int, seed: int | None = None) -> EngineParams:
    """CKKS parameters of BASELINE.json configs 1-5."""
    table = {
        1: dict(slots=1 << 12, delta=40, prime_bits=(60, 40)),
        2: dict(slots=1 << 13, delta=40, prime_bits=(60, 40, 40, 40, 40)),
        3: dict(slots=1 << 13, delta=40, prime_bits=(60, 40, 40, 40, 40, 40)),
        4: dict(slots=1 << 14, delta=45, prime_bits=(60,) + (45,) * 7),
        5: dict(slots=1 << 14, delta=45, prime_bits=(60,) + (45,) * 7),
    }
    if cfg not in table:
        raise EngineError(f"unknown config {cfg}")
    kw = dict(table[cfg])
    kw["seed"] = cfg - 1 if seed is None else seed
    return EngineParams(**kw)
