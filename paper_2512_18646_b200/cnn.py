"""Encrypted CNN layers on column ciphertexts (BASELINE configs 3, 4, 5b).

The reference has the building blocks (encode_image_columns, conv_columns,
poly_activation; multicipher.py:106-172, pipeline.py:180-197) but no
multi-channel layer, padding or stride.  ``conv_layer``
composes them the way the paper describes (channel sum):
host zero padding, one conv_columns_multi driver call for every
(filter, channel, tap), stride-2 layers computing only the even output
columns (even rows are selected at decode), and one batched activation over
every output ciphertext.
"""

from __future__ import annotations

import numpy as np

from .engine import CkksEngine, EngineError
from .multicipher import ColumnEncodedImage, conv_columns_multi, encode_image_columns, pad_images
from .pipeline import poly_activation_batch

__all__ = ["encode_images", "conv_layer", "decode_layer", "square_batch"]


def encode_images(engine: CkksEngine, images, padding: int = 0) -> list[ColumnEncodedImage]:
    """images (m, C, h, w) -> one ColumnEncodedImage per channel (w column ciphertexts each)."""
    arr = np.asarray(images, dtype=np.float64)
    if arr.ndim != 4:
        raise EngineError(f"expected (m, C, h, w) images, got shape {arr.shape}")
    if padding:
        arr = pad_images(arr, padding)
    return [encode_image_columns(engine, arr[:, c]) for c in range(arr.shape[1])]


def conv_layer(engine: CkksEngine, chans, weights, bias=None, stride: int = 1, activation=None) -> list[ColumnEncodedImage]:
    """Multi-channel convolution (+ optional polynomial activation) of encrypted column images.

    ``weights`` [F][C][k][k]; ``activation`` = 4 coefficients (c0..c3) or None.  With
    stride s only every s-th output column is computed; rows are subsampled by
    ``decode_layer`` (the column layout keeps all rows of a column in one ciphertext).
    """
    w = np.asarray(weights, dtype=np.float64)
    F = w.shape[0]
    bias = np.zeros(F) if bias is None else np.asarray(bias, dtype=np.float64)
    base = chans[0]
    out_w = base.w - w.shape[-1] + 1
    cols = list(range(0, out_w, stride))
    ys = conv_columns_multi(engine, chans, w, bias, out_cols=cols)
    if activation is None:
        return ys
    flat = [ct for y in ys for ct in y.cts]
    act = poly_activation_batch(engine, flat, activation)
    out, pos = [], 0
    for y in ys:
        n = len(y.cts)
        out.append(ColumnEncodedImage(act[pos: pos + n], y.h, y.w, y.m, y.stride))
        pos += n
    return out


def square_batch(engine: CkksEngine, cts):
    """x -> x^2 for many ciphertexts (one level): the square activation of config 3."""
    from . import _lib
    import torch

    cts = list(cts)
    lv = min(c.level for c in cts)
    cts = [engine.adjust(c, lv) for c in cts]
    out = torch.empty((len(cts), 2, lv, engine.N), dtype=torch.int64, device=engine.device)
    ptrs = _lib.ptr_array([c.ptr() for c in cts])
    _lib.check(engine._lib.vr_mul(engine.handle, ptrs, ptrs, _lib.ptr_array([out[i].data_ptr() for i in range(len(cts))]),
                                  len(cts), lv))
    from .engine import Ciphertext

    res = []
    for i, c in enumerate(cts):
        engine._meter.mul_count += 1
        engine._observe(c.depth + 1)
        res.append(Ciphertext(out[i], lv - 1, engine.scales[lv - 1], c.depth + 1, c.layout, engine._id))
    return res


def decode_layer(engine: CkksEngine, ys, stride: int = 1) -> np.ndarray:
    """Decrypt a conv layer's output to (m, F, out_h, out_w) (rows subsampled by ``stride``)."""
    outs = []
    for y in ys:
        vecs = engine.dec_batch(y.cts)  # [w][slots]
        img = np.stack([vecs[:, b * y.stride: b * y.stride + y.h].T for b in range(y.m)])  # (m, h, w)
        outs.append(img[:, ::stride, :])
    return np.stack(outs, axis=1)
