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

from dataclasses import dataclass

import numpy as np

from .engine import CkksEngine, EngineError
from .multicipher import ColumnEncodedImage, conv_columns_multi, encode_image_columns, pad_images
from .pipeline import poly_activation_batch

__all__ = ["encode_images", "conv_layer", "decode_layer", "square_batch", "encode_cfg3_model", "cnn_cfg3", "decode_logits",
           "dense_columns", "block_sum", "rotate_batch"]


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
    _lib.check(engine._lib.vr_mul(engine.handle, ptrs, ptrs, _lib.row_ptrs(out, len(cts)),
                                  len(cts), lv))
    from .engine import Ciphertext

    res = []
    for i, c in enumerate(cts):
        engine._meter.mul_count += 1
        engine._observe(c.depth + 1)
        res.append(Ciphertext.at(out, i, lv - 1, engine.scales[lv - 1], c.depth + 1, c.layout, engine._id))
    return res


def decode_layer(engine: CkksEngine, ys, stride: int = 1) -> np.ndarray:
    """Decrypt a conv layer's output to (m, F, out_h, out_w) (rows subsampled by ``stride``)."""
    outs = []
    for y in ys:
        # only the valid slots (b * stride + i, i < h) leave the device: [w][m * h]
        sel = (np.arange(y.m)[:, None] * y.stride + np.arange(y.h)[None, :]).reshape(-1)
        vecs = engine.dec_batch(y.cts, select=sel)
        img = vecs.reshape(len(y.cts), y.m, y.h).transpose(1, 2, 0)  # (m, h, w)
        outs.append(img[:, ::stride, :])
    return np.stack(outs, axis=1)


# ---------------------------------------------------------------------------
# Config 3: conv 5x4x4 stride 2 -> square -> dense 845->64 -> square -> dense 64->10
# entirely in the column layout (the reference has no column-layout dense layer,
# SURVEY.md section 8d).  Depth 1 + 1 + 1 + 1 + 1 = 5.

def encode_plain_batch(engine: CkksEngine, rows, level: int, scale: float):
    """Encode many slot vectors as plaintexts [count][level+1][N] (one launch)."""
    import torch

    from . import _lib

    vals = engine._pad(rows)
    d_vals = engine._h2d(vals)
    pts = torch.empty((vals.shape[0], level + 1, engine.N), dtype=torch.int64, device=engine.device)
    _lib.check(engine._lib.vr_encode(engine.handle, d_vals.data_ptr(), vals.shape[0], vals.shape[1], level, scale,
                                     pts.data_ptr()))
    return pts


def dense_columns(engine: CkksEngine, cts, pts, ny: int):
    """Y[u] = sum_j pts[u*nx + j] (.) cts[j], rescaled: a plaintext-weight dense layer.

    Metered like the reference composition: nx cmuls and nx-1 adds per output.
    """
    import torch

    from . import _lib
    from .engine import Ciphertext

    cts = list(cts)
    nx = len(cts)
    lv = cts[0].level
    if any(c.level != lv for c in cts):
        raise EngineError("dense_columns inputs must share a level")
    out = torch.empty((ny, 2, lv, engine.N), dtype=torch.int64, device=engine.device)
    _lib.check(engine._lib.vr_pt_matvec(engine.handle, _lib.ptr_array([c.ptr() for c in cts]), nx,
                                        _lib.row_ptrs(pts, ny * nx), ny, lv,
                                        _lib.row_ptrs(out, ny)))
    depth = max(c.depth for c in cts) + 1
    engine._meter.cmul_count += ny * nx
    engine._meter.add_count += ny * (nx - 1)
    engine._observe(depth)
    return [Ciphertext.at(out, u, lv - 1, engine.scales[lv - 1], depth, cts[0].layout, engine._id) for u in range(ny)]


def rotate_batch(engine: CkksEngine, cts, steps):
    """Hoisted rotations of many ciphertexts: result[c][r] = rot(cts[c], steps[r])."""
    import ctypes

    import torch

    from . import _lib
    from .engine import Ciphertext

    cts = list(cts)
    lv = cts[0].level
    steps = [int(s) for s in steps]
    nr = len(steps)
    flat = torch.empty((len(cts) * nr, 2, lv + 1, engine.N), dtype=torch.int64, device=engine.device)
    st = (ctypes.c_int64 * nr)(*steps)
    _lib.check(engine._lib.vr_rotate(engine.handle, _lib.ptr_array([c.ptr() for c in cts]), _lib.row_ptrs(flat),
                                     len(cts), lv, nr, st))
    engine._meter.rot_count += len(cts) * nr
    return [[Ciphertext.at(flat, i * nr + r, lv, c.scale, c.depth, c.layout, engine._id) for r in range(nr)]
            for i, c in enumerate(cts)]


def add_batch(engine: CkksEngine, xs, ys):
    import torch

    from . import _lib
    from .engine import Ciphertext

    xs, ys = list(xs), list(ys)
    lv = xs[0].level
    out = torch.empty((len(xs), 2, lv + 1, engine.N), dtype=torch.int64, device=engine.device)
    _lib.check(engine._lib.vr_add(engine.handle, _lib.ptr_array([x.ptr() for x in xs]), _lib.ptr_array([y.ptr() for y in ys]),
                                  _lib.row_ptrs(out, len(xs)), len(xs), 1, lv, 0))
    engine._meter.add_count += len(xs)
    return [Ciphertext.at(out, i, lv, x.scale, max(x.depth, y.depth), x.layout, engine._id) for i, (x, y) in enumerate(zip(xs, ys))]


def block_sum(engine: CkksEngine, cts, terms: int, stride: int):
    """slot p <- sum_{r < terms} slot(p + stride * r), by rotate-and-add doubling (hoisted per level).

    For terms = 13, stride = 2 this uses 5 rotations: T2 = T1 + rot(T1, 2), T4 = T2 + rot(T2, 4),
    T8 = T4 + rot(T4, 8), total = T8 + rot(T4, 16) + rot(T1, 24).
    """
    bits = [b for b in range(terms.bit_length()) if terms >> b & 1]
    top = terms.bit_length() - 1
    T = {0: list(cts)}
    # extra rotations each power needs for the final combination (offset = stride * higher bits)
    offsets = {}
    acc_off = 1 << top
    for b in sorted(bits, reverse=True)[1:]:
        offsets[b] = stride * acc_off
        acc_off += 1 << b
    for lvl in range(top + 1):
        steps = []
        if lvl < top:
            steps.append(stride << lvl)
        if lvl in offsets:
            steps.append(offsets[lvl])
        rot = rotate_batch(engine, T[lvl], steps) if steps else [[] for _ in T[lvl]]
        if lvl < top:
            T[lvl + 1] = add_batch(engine, T[lvl], [r[0] for r in rot])
        if lvl in offsets:
            offsets[lvl] = [r[-1] for r in rot]
    total = T[top]
    for b in sorted(offsets):
        total = add_batch(engine, total, offsets[b])
    return total


@dataclass(frozen=True, eq=False)
class Cfg3Model:
    """Plaintext-encoded dense layers of config 3 (the provider encodes the model once, like the
    reference's encode_model, pipeline.py:339-372)."""

    w: np.ndarray
    pts1: object  # [ny * F * no][level+1][N] plaintexts of W1 at the dense-1 input level
    pts2: object  # [nz * ny][level+1][N] constant plaintexts of W2
    m: int
    h: int
    ny: int
    nz: int


def encode_cfg3_model(engine: CkksEngine, w, w1, w2, m: int = 64, h: int = 28) -> Cfg3Model:
    """Encode config 3's dense weights as plaintexts at the levels the network reaches them."""
    F, _, k, _ = w.shape
    out_w = h - k + 1
    nr = no = len(range(0, out_w, 2))
    L = engine.L
    lv1, lv2 = L - 2, L - 4  # after conv + square / after dense 1 + square
    S = engine.slots
    ny, nz = w1.shape[0], w2.shape[0]
    rows = list(range(0, h - k + 1, 2))
    masks = np.zeros((ny, F * no, S))
    slot_idx = (np.arange(m)[:, None] * h + np.asarray(rows)[None, :]).reshape(-1)  # (b, r) -> slot
    for f in range(F):
        for o in range(no):
            wv = w1[:, f * nr * no + np.arange(nr) * no + o]  # (ny, nr): W1[u, f*169 + r*13 + o]
            masks[:, f * no + o, slot_idx] = np.tile(wv, (1, m))
    pts1 = encode_plain_batch(engine, masks.reshape(ny * F * no, S), lv1, engine.scales[lv1])
    pts2 = encode_plain_batch(engine, np.repeat(np.asarray(w2).reshape(-1, 1), S, axis=1), lv2, engine.scales[lv2])
    return Cfg3Model(np.asarray(w, dtype=np.float64), pts1, pts2, m, h, ny, nz)


def cnn_cfg3(engine: CkksEngine, imgs, w, w1=None, w2=None, model: Cfg3Model | None = None):
    """Config 3 on a batch of (m, 28, 28) images: returns the 10 logit ciphertexts (logit v of
    image b at slot b*28).  Pass a pre-encoded ``model`` to skip encoding the dense weights."""
    imgs = np.asarray(imgs, dtype=np.float64)
    m, h, wd = imgs.shape
    if model is None:
        model = encode_cfg3_model(engine, w, w1, w2, m, h)
    w = model.w
    F, _, k, _ = w.shape
    cols = list(range(0, wd - k + 1, 2))  # stride-2 columns: 13
    x = encode_image_columns(engine, imgs)
    conv = conv_columns_multi(engine, [x], w, np.zeros(F), out_cols=cols)
    feats = square_batch(engine, [ct for y in conv for ct in y.cts])  # F*13 cts, order (f, o)
    hid = dense_columns(engine, feats, model.pts1, model.ny)
    hid = block_sum(engine, hid, len(cols), 2)
    hid = square_batch(engine, hid)
    return dense_columns(engine, hid, model.pts2, model.nz)


def decode_logits(engine: CkksEngine, logits, m: int, stride: int) -> np.ndarray:
    vecs = engine.dec_batch(logits)  # [10][S]
    return vecs[:, np.arange(m) * stride].T
