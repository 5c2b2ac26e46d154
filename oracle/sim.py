"""Numpy restatement of the reference's column-ciphertext path (exact float64
slot simulator).  TEST INFRASTRUCTURE ONLY -- the decoded-value oracle.

Follows /root/reference/pkg/src/packedhe:
  SimEngine.enc/dec/add/mul/cmul/rot/mask   engine.py:193-251
  Meter (add/mul/cmul/rot/enc, max depth)    engine.py:93-131
  encode_left / encode_right / matmul_outer  multicipher.py:62-103
  encode_image_columns / conv_columns /
  reassemble_columns                         multicipher.py:106-172
  poly_activation                            pipeline.py:180-197
  oracle_matmul / oracle_conv / oracle_poly  oracle.py:19-56
Pinned against fixtures produced by the reference itself
(tests/golden/make_golden.py -> tests/golden/reference_golden.npz).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


class SimError(ValueError):
    pass


@dataclass
class SimMeter:
    add_count: int = 0
    mul_count: int = 0
    cmul_count: int = 0
    rot_count: int = 0
    enc_count: int = 0
    max_depth: int = 0


@dataclass
class SimCt:
    slots: np.ndarray
    depth: int = 0


class SimEngine:
    def __init__(self, slots: int):
        self.slots = slots
        self.meter = SimMeter()

    def _obs(self, d):
        self.meter.max_depth = max(self.meter.max_depth, d)

    def enc(self, values) -> SimCt:  # engine.py:193-202
        v = np.asarray(values, dtype=np.float64).reshape(-1)
        if v.size > self.slots:
            raise SimError("capacity")
        full = np.zeros(self.slots)
        full[: v.size] = v
        self.meter.enc_count += 1
        self._obs(0)
        return SimCt(full, 0)

    def dec(self, ct: SimCt) -> np.ndarray:  # engine.py:204-206
        return ct.slots.copy()

    def add(self, a, b):  # engine.py:208-213
        d = max(a.depth, b.depth)
        self.meter.add_count += 1
        self._obs(d)
        return SimCt(a.slots + b.slots, d)

    def mul(self, a, b):  # engine.py:215-220
        d = max(a.depth, b.depth) + 1
        self.meter.mul_count += 1
        self._obs(d)
        return SimCt(a.slots * b.slots, d)

    def cmul(self, mask: np.ndarray, ct):  # engine.py:222-230
        self.meter.cmul_count += 1
        self._obs(ct.depth + 1)
        return SimCt(np.asarray(mask) * ct.slots, ct.depth + 1)

    def rot(self, ct, l: int):  # engine.py:232-236
        self.meter.rot_count += 1
        self._obs(ct.depth)
        return SimCt(np.roll(ct.slots, -l), ct.depth)

    def mask(self, values) -> np.ndarray:  # engine.py:244-251
        v = np.asarray(values, dtype=np.float64).reshape(-1)
        full = np.zeros(self.slots)
        full[: v.size] = v
        return full


def encode_left(eng, a, p):  # multicipher.py:62-72
    a = np.atleast_2d(np.asarray(a, dtype=np.float64))
    m, n = a.shape
    if m * p > eng.slots:
        raise SimError("capacity")
    return [eng.enc(np.repeat(a[:, k], p)) for k in range(n)]


def encode_right(eng, b, m):  # multicipher.py:75-85
    b = np.atleast_2d(np.asarray(b, dtype=np.float64))
    n, p = b.shape
    if m * p > eng.slots:
        raise SimError("capacity")
    return [eng.enc(np.tile(b[k, :], m)) for k in range(n)]


def matmul_outer(eng, left, right, m, p):  # multicipher.py:88-103
    acc = None
    for lk, rk in zip(left, right):
        term = eng.mul(lk, rk)
        acc = term if acc is None else eng.add(acc, term)
    return eng.dec(acc)[: m * p].reshape(m, p), acc


def encode_image_columns(eng, images):  # multicipher.py:106-120
    arr = np.asarray(images, dtype=np.float64)
    if arr.ndim == 2:
        arr = arr[None]
    m, h, w = arr.shape
    if m * h > eng.slots:
        raise SimError("capacity")
    return [eng.enc(arr[:, :, j].reshape(-1)) for j in range(w)], (h, w, m, h)


def conv_columns(eng, cts, geom, weights, bias):  # multicipher.py:123-162
    h, w, m, stride = geom
    weights = np.asarray(weights, dtype=np.float64)
    k = weights.shape[0]
    out_h, out_w = h - k + 1, w - k + 1
    valid = np.zeros((m, stride))
    valid[:, :out_h] = 1.0
    valid = valid.reshape(-1)
    rotated = {}

    def shifted(j, p):
        if p == 0:
            return cts[j]
        if (j, p) not in rotated:
            rotated[(j, p)] = eng.rot(cts[j], p)
        return rotated[(j, p)]

    out = []
    for jp in range(out_w):
        b = np.zeros((m, stride))
        b[:, :out_h] = bias
        acc = eng.enc(b.reshape(-1))
        for q in range(k):
            for p in range(k):
                wgt = weights[p, q]
                if wgt == 0.0:
                    continue
                acc = eng.add(acc, eng.cmul(eng.mask(wgt * valid), shifted(jp + q, p)))
        out.append(acc)
    return out, (out_h, out_w, m, stride)


def reassemble_columns(eng, cts, geom):  # multicipher.py:165-172
    h, w, m, stride = geom
    out = np.empty((m, h, w))
    for j, ct in enumerate(cts):
        vec = eng.dec(ct)
        for b in range(m):
            out[b, :, j] = vec[b * stride: b * stride + h]
    return out


def poly_activation(eng, ct, coeffs):  # pipeline.py:180-197
    c0, c1, c2, c3 = (float(c) for c in coeffs)
    s = eng.slots
    x2 = eng.mul(ct, ct)
    inner = eng.add(eng.cmul(eng.mask(np.full(s, c3)), ct), eng.enc(np.full(s, c2)))
    out = eng.mul(x2, inner)
    out = eng.add(out, eng.cmul(eng.mask(np.full(s, c1)), ct))
    return eng.add(out, eng.enc(np.full(s, c0)))


def oracle_matmul(a, b):  # oracle.py:19-34
    a = np.atleast_2d(np.asarray(a, dtype=np.float64))
    b = np.atleast_2d(np.asarray(b, dtype=np.float64))
    m, n = a.shape
    n2, p = b.shape
    if n != n2:
        raise ValueError("inner dims differ")
    out = np.zeros((m, p))
    for i in range(m):
        for j in range(p):
            s = 0.0
            for k in range(n):
                s += a[i, k] * b[k, j]
            out[i, j] = s
    return out


def oracle_conv(image, weights, bias=0.0):  # oracle.py:37-49
    image = np.asarray(image, dtype=np.float64)
    weights = np.asarray(weights, dtype=np.float64)
    h, w = image.shape
    k = weights.shape[0]
    out = np.zeros((h - k + 1, w - k + 1))
    for i in range(h - k + 1):
        for j in range(w - k + 1):
            out[i, j] = bias + float(np.sum(image[i: i + k, j: j + k] * weights))
    return out


def oracle_poly(x, coeffs):  # oracle.py:52-56
    x = np.asarray(x, dtype=np.float64)
    c0, c1, c2, c3 = (float(c) for c in coeffs)
    return c0 + c1 * x + c2 * x * x + c3 * x * x * x


def oracle_flatten(maps):  # oracle.py:59-61
    return np.concatenate([np.asarray(m, dtype=np.float64).reshape(-1) for m in maps])


def oracle_forward(weights, images):  # oracle.py:64-82
    """Plaintext conv -> act -> flatten -> fc -> act -> fc of the Table-1 CNN."""
    images = np.asarray(images, dtype=np.float64)
    out = []
    for img in images:
        maps = [oracle_poly(conv_fast(img[None], k.weights, k.bias)[0], weights.act1) for k in weights.conv_kernels]
        h1 = oracle_poly(np.asarray(weights.fc1_weight) @ oracle_flatten(maps) + weights.fc1_bias, weights.act2)
        out.append(np.asarray(weights.fc2_weight) @ h1 + weights.fc2_bias)
    return np.stack(out)


def table1_weights(seed: int):
    """Seeded Table-1 model in the reference suite's distribution (test_pipeline.py:32-46);
    returns plain arrays: (kernels [4][3][3], kernel biases [4], fc1_w, fc1_b, fc2_w, fc2_b)."""
    rng = np.random.default_rng(seed)
    kw, kb = [], []
    for _ in range(4):
        kw.append(rng.uniform(-0.4, 0.4, size=(3, 3)))
        kb.append(float(rng.uniform(-0.1, 0.1)))
    fc1_w = rng.uniform(-0.05, 0.05, size=(64, 2704))
    fc1_b = rng.uniform(-0.1, 0.1, size=64)
    fc2_w = rng.uniform(-0.3, 0.3, size=(10, 64))
    fc2_b = rng.uniform(-0.1, 0.1, size=10)
    return np.array(kw), np.array(kb), fc1_w, fc1_b, fc2_w, fc2_b


def conv_fast(images, weights, bias=0.0):
    """Vectorised valid conv for large fixtures (same values as oracle_conv up to fp reassociation)."""
    images = np.asarray(images, dtype=np.float64)
    w = np.asarray(weights, dtype=np.float64)
    k = w.shape[-1]
    m, h, wd = images.shape
    out = np.full((m, h - k + 1, wd - k + 1), float(bias))
    for p in range(k):
        for q in range(k):
            out += w[p, q] * images[:, p: p + h - k + 1, q: q + wd - k + 1]
    return out
