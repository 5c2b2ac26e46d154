"""OracleEngine: CPU restatement of the engine policy on top of the C residue
oracle (oracle/ckks_oracle.c).  TEST INFRASTRUCTURE ONLY.

It follows the reference SlotEngine surface (engine.py:193-251) and makes the
same level/scale decisions as the GPU engine, written
independently here so that tests can demand bit-identical residues from the
GPU for the same seed, nonces and inputs.  Ciphertexts are plain numpy uint64
arrays [deg+1][level+1][N] with (level, scale, depth) carried alongside.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .ckks import OracleCkks, gen_primes


@dataclass
class OCt:
    data: np.ndarray
    level: int
    scale: float
    depth: int = 0
    layout: tuple | None = None


class OracleEngine:
    def __init__(self, slots: int, prime_bits, special_bits: int = 60, delta: int = 45, delta_c: int = 20,
                 seed: int = 0, encryption: str = "secret"):
        self.slots = slots
        self.log_n = int(math.log2(2 * slots))
        self.N = 2 * slots
        self.delta = delta
        self.delta_c = delta_c
        self.q = [int(x) for x in gen_primes(self.log_n, list(prime_bits) + [special_bits])]
        self.L = len(prime_bits) - 1
        self.c = OracleCkks(self.log_n, self.q, seed, sym_enc=(encryption == "secret"))
        s = [0.0] * (self.L + 1)
        s[self.L] = float(2 ** delta)
        for lv in range(self.L, 0, -1):
            s[lv - 1] = (s[lv] * s[lv]) / float(self.q[lv])
        self.scales = s
        self.nonce = 0

    @classmethod
    def from_params(cls, p):
        """Build from a product EngineParams-like object (only plain fields are read)."""
        return cls(p.slots, p.prime_bits, p.special_bits, p.delta, p.delta_c, p.seed, p.encryption)

    # -- primitives ------------------------------------------------------
    def enc(self, values, layout=None) -> OCt:
        v = np.asarray(values, dtype=np.float64).reshape(-1)
        ct = self.c.encrypt(v, self.L, self.scales[self.L], self.nonce)
        self.nonce += 1
        return OCt(ct, self.L, self.scales[self.L], 0, layout)

    def dec(self, ct: OCt) -> np.ndarray:
        return self.c.decrypt_decode(ct.data, ct.scale)

    def adjust(self, ct: OCt, level: int) -> OCt:
        if level == ct.level:
            return ct
        data = ct.data
        if ct.level > level + 1:
            data = self.c.drop_level(data, level + 1)
        k = int(round(self.scales[level] * float(self.q[level + 1]) / ct.scale))
        data = self.c.rescale(self.c.mul_scalar(data, k))
        return OCt(data, level, self.scales[level], ct.depth, ct.layout)

    def _align(self, a: OCt, b: OCt):
        if a.level == b.level:
            return a, b
        lv = min(a.level, b.level)
        return self.adjust(a, lv), self.adjust(b, lv)

    def add(self, a: OCt, b: OCt) -> OCt:
        a, b = self._align(a, b)
        return OCt(self.c.add(a.data, b.data), a.level, self.scales[a.level], max(a.depth, b.depth), a.layout)

    def mul(self, a: OCt, b: OCt) -> OCt:
        a, b = self._align(a, b)
        lv = a.level
        return OCt(self.c.mul(a.data, b.data), lv - 1, self.scales[lv - 1], max(a.depth, b.depth) + 1, a.layout)

    def mask(self, values, role: str = "constant") -> np.ndarray:
        """Zero-padded slot vector (engine.py:244-251); cmul accepts it or a PlainMask-like object."""
        vec = np.asarray(values, dtype=np.float64).reshape(-1)
        full = np.zeros(self.slots)
        full[: vec.size] = vec
        return full

    def cmul(self, values, ct: OCt) -> OCt:
        vals = np.asarray(getattr(values, "values", values), dtype=np.float64).reshape(-1)
        lv = ct.level
        if np.all(vals == vals[0]):
            tmp = self.c.mul_scalar(ct.data, int(round(float(vals[0]) * ct.scale)))
        else:
            tmp = self.c.mul_plain(ct.data, self.c.encode(vals, lv, ct.scale))
        return OCt(self.c.rescale(tmp), lv - 1, self.scales[lv - 1], ct.depth + 1, ct.layout)

    def rot(self, ct: OCt, l: int) -> OCt:
        if int(l) % self.slots == 0:
            return OCt(ct.data, ct.level, ct.scale, ct.depth, ct.layout)
        return OCt(self.c.rotate(ct.data, int(l)), ct.level, ct.scale, ct.depth, ct.layout)

    # -- the batched surface of the product engine (CkksEngine.*_batch), as plain loops --------
    # The product's algorithm modules (matmul.py, conv.py, virtual.py, pipeline.py) drive only this
    # surface; these loops are the per-op definition the GPU's batched launches must reproduce.
    def enc_batch(self, rows, layout=None, nonce0=None):
        if nonce0 is None:
            return [self.enc(r, layout) for r in rows]
        saved, self.nonce = self.nonce, int(nonce0)  # explicit nonces leave the running counter alone
        try:
            return [self.enc(r, layout) for r in rows]
        finally:
            self.nonce = saved

    def rot_batch(self, cts, steps):
        return [[self.rot(c, s) for s in steps] for c in cts]

    def add_batch(self, xs, ys):
        return [self.add(x, y) for x, y in zip(xs, ys)]

    def mul_batch(self, xs, ys):
        return [self.mul(x, y) for x, y in zip(xs, ys)]

    def cmul_batch(self, masks, cts):
        cts = list(cts)
        if not isinstance(masks, (list, tuple)):
            masks = [masks] * len(cts)
        return [self.cmul(m, c) for m, c in zip(masks, cts)]

    def sum_batch(self, acc, cts):
        for c in cts:
            acc = self.add(acc, c)
        return acc

    # -- fused drivers (same op order as the CUDA drivers) -----------------
    def matmul_outer_blocks(self, lefts, rights):
        """lefts: list of lists of OCt (row blocks), rights: list of OCt."""
        allc = [c for lf in lefts for c in lf] + list(rights)
        lv = min(c.level for c in allc)
        allc = [self.adjust(c, lv) for c in allc]
        n = len(rights)
        R = [c.data for c in allc[len(allc) - n:]]
        outs = []
        for b in range(len(lefts)):
            Lb = [c.data for c in allc[b * n:(b + 1) * n]]
            outs.append(OCt(self.c.matmul_outer(Lb, R), lv - 1, self.scales[lv - 1]))
        return outs

    def conv_columns_multi(self, X, C, W, weights, biases, out_cols, m, stride, out_h):
        """X: list of C*W OCt; weights [F][C][k][k] floats; mirrors multicipher.conv_columns_multi."""
        lv = min(c.level for c in X)
        X = [self.adjust(c, lv) for c in X]
        w = np.asarray(weights, dtype=np.float64)
        F, _, k, _ = w.shape
        dc = float(2 ** self.delta_c)
        w_int = np.array([int(round(float(x) * dc)) for x in w.reshape(-1)], dtype=np.int64).reshape(w.shape)
        scale = X[0].scale
        b_ints = [int(round(float(b) * scale * dc)) for b in np.broadcast_to(np.asarray(biases, dtype=np.float64).reshape(-1), (F,))]
        b_res = np.array([[bi % self.q[i] for i in range(lv + 1)] for bi in b_ints], dtype=np.uint64)
        valid = np.zeros((m, stride))
        valid[:, :out_h] = 1.0
        mask_pt = self.c.encode(valid.reshape(-1), lv, self.scales[lv] / dc)
        Y = self.c.conv_columns([x.data for x in X], C, W, k, w_int, b_res, F, list(out_cols), mask_pt)
        return [OCt(y, lv - 1, self.scales[lv - 1]) for y in Y]

    def poly_activation(self, ct: OCt, coeffs) -> OCt:
        lv = ct.level
        c0, c1, c2, c3 = (float(c) for c in coeffs)
        s, q = self.scales, self.q
        kc = (int(round(c3 * s[lv])), int(round(c2 * s[lv - 1])),
              int(round(c1 * s[lv - 1] * s[lv - 1] / s[lv])), int(round(c0 * s[lv - 2])))
        out = self.c.poly_activation(ct.data, kc, c3 == 0.0)
        return OCt(out, lv - 2, s[lv - 2], ct.depth + 2, ct.layout)
