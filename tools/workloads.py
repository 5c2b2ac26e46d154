"""Seeded synthetic inputs of BASELINE.json configs 1-5 and their plaintext results.

Draw order follows SURVEY.md section 8d: rng = default_rng(seed) (the PCG64
generator the reference tests use), data drawn first in the listed order.
BASELINE.json names no public dataset; everything here is synthetic.
"""

from __future__ import annotations

import numpy as np

ACT4 = (0.25, 0.5, 0.125, 0.0)  # 0.125 x^2 + 0.5 x + 0.25 (config 4)


def cfg_matmul(cfg: int):
    dim = {1: 8, 2: 64, 5: 256}[cfg]
    rng = np.random.default_rng({1: 0, 2: 1, 5: 4}[cfg])
    a = rng.uniform(-1, 1, (dim, dim))
    b = rng.uniform(-1, 1, (dim, dim))
    return a, b


def cfg4(images: int = 16, seed: int = 3):
    rng = np.random.default_rng(seed)
    imgs = rng.uniform(0, 1, (images, 3, 224, 224))
    w = rng.normal(0, 0.05, (16, 3, 3, 3))
    return imgs, w, np.zeros(16)


def cfg5b(images: int = 512):
    return cfg4(images=images, seed=4)


def cfg3():
    rng = np.random.default_rng(2)
    imgs = rng.uniform(0, 1, (64, 28, 28))
    w = rng.normal(0, 0.1, (5, 1, 4, 4))
    w1 = rng.normal(0, 0.1, (64, 845))
    w2 = rng.normal(0, 0.1, (10, 64))
    return imgs, w, w1, w2


def conv_plain(images, w, bias, padding=0, stride=1):
    """(m, C, h, w) * (F, C, k, k) -> (m, F, oh, ow), cross-correlation like oracle_conv (oracle.py:37-49)."""
    x = np.asarray(images, dtype=np.float64)
    if padding:
        x = np.pad(x, ((0, 0), (0, 0), (padding, padding), (padding, padding)))
    m, C, h, wd = x.shape
    F, _, k, _ = w.shape
    oh, ow = h - k + 1, wd - k + 1
    out = np.zeros((m, F, oh, ow))
    for f in range(F):
        acc = np.full((m, oh, ow), float(bias[f]))
        for c in range(C):
            for p in range(k):
                for q in range(k):
                    acc += w[f, c, p, q] * x[:, c, p: p + oh, q: q + ow]
        out[:, f] = acc
    return out[:, :, ::stride, ::stride]


def poly_plain(x, coeffs):
    c0, c1, c2, c3 = coeffs
    return c0 + c1 * x + c2 * x * x + c3 * x * x * x


def cfg3_plain(imgs, w, w1, w2):
    """conv 5x4x4 stride 2 -> square -> dense 845->64 -> square -> dense 64->10 (map-major flatten)."""
    y = conv_plain(imgs[:, None], w, np.zeros(5), stride=2)  # (64, 5, 13, 13)
    y = y * y
    flat = y.reshape(y.shape[0], -1)  # index f*169 + r*13 + o
    h = flat @ w1.T
    h = h * h
    return h @ w2.T
