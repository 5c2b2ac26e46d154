"""Multi-ciphertext encodings and their batched GPU evaluation.

Same public names, signatures, validation and meter accounting as the
reference (multicipher.py:23-172):

* ``encode_left`` / ``encode_right``   n column ciphertexts per operand, all
  encrypted in ONE launch (multicipher.py:62-85);
* ``matmul_outer``   sum_k L_k * R_k as one fused tensor-sum kernel, then a
  single relinearisation and rescale (multicipher.py:88-103);
* ``encode_image_columns`` / ``conv_columns`` / ``reassemble_columns``
  (multicipher.py:106-172): hoisted rotations shared by every tap, one MAC
  kernel for all output columns.

Extensions the BASELINE configs need and the reference lacks (SURVEY.md
section 8d): ``conv_columns_multi`` (C input channels x F filters, the
paper's channel sum, with an explicit output-column list so a
stride-2 layer computes only even columns), ``matmul_outer_blocks`` (row-tiled
left operand sharing one right operand) and ``pad_images``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .encoding import Encoding, Kernel, MatrixShape, PackedMatrix
from .engine import CapacityError, Ciphertext, CkksEngine, CtBatch, EngineError, LayoutError

__all__ = [
    "ColumnEncodedMatrix",
    "ColumnEncodedImage",
    "encode_left",
    "encode_right",
    "matmul_outer",
    "matmul_outer_blocks",
    "matmul_outer_many",
    "encode_image_columns",
    "conv_columns",
    "conv_columns_multi",
    "reassemble_columns",
    "pad_images",
    "conv_constants",
]


@dataclass(frozen=True, eq=False)
class ColumnEncodedMatrix:
    """n ciphertexts holding one matmul operand in broadcast form."""

    cts: list
    role: str  # "left" or "right"
    m: int
    n: int
    p: int


@dataclass(frozen=True, eq=False)
class ColumnEncodedImage:
    """w ciphertexts, one image column each; batched images stack at ``stride``."""

    cts: list
    h: int
    w: int
    m: int
    stride: int


def encode_left(engine: CkksEngine, a, p: int) -> ColumnEncodedMatrix:
    """Ciphertext k = column k of A broadcast across an m x p grid (slot i*p+j = A[i,k])."""
    a = np.atleast_2d(np.asarray(a, dtype=np.float64))
    m, n = a.shape
    if m * p > engine.slots:
        raise CapacityError(f"{m}x{p} broadcast needs {m * p} slots, engine has {engine.slots}")
    # ct k, slot i*p + j = A[i, k]: broadcast done on the device from the raw m x n matrix
    cts = engine.enc_strided(a, count=n, nvals=m * p, p=p, sc=1, s1=n, s2=0, layout=("grid", m, p))
    return _fresh(engine, ColumnEncodedMatrix(cts, "left", m, n, p))


def encode_right(engine: CkksEngine, b, m: int) -> ColumnEncodedMatrix:
    """Ciphertext k = row k of B tiled down m grid rows (slot i*p+j = B[k,j])."""
    b = np.atleast_2d(np.asarray(b, dtype=np.float64))
    n, p = b.shape
    if m * p > engine.slots:
        raise CapacityError(f"{m}x{p} tiling needs {m * p} slots, engine has {engine.slots}")
    # ct k, slot i*p + j = B[k, j]: tiling done on the device from the raw n x p matrix
    cts = engine.enc_strided(b, count=n, nvals=m * p, p=p, sc=p, s1=0, s2=1, layout=("grid", m, p))
    return _fresh(engine, ColumnEncodedMatrix(cts, "right", m, n, p))


class _OperandCache:
    """Validated view of a column-encoded operand for one engine: level, max depth, the storage
    tensors, and the device pointer table -- kept as a uint64 numpy array; the ctypes array the
    C-ABI takes and the Python list are made from it on first use."""

    __slots__ = ("eid", "level", "depth", "storages", "_np", "_arr", "_list")

    def __init__(self, eid, level, depth, storages, np_ptrs=None, ptrs=None):
        self.eid, self.level, self.depth, self.storages = eid, level, depth, storages
        self._np = np_ptrs if np_ptrs is not None else np.array(ptrs, dtype=np.uint64)
        self._arr = None
        self._list = ptrs

    @property
    def arr(self):
        a = self._arr
        if a is None:
            a = self._arr = (ctypes.c_void_p * max(1, self._np.size)).from_buffer(self._np) if self._np.size else _lib.ptr_array([])
        return a

    @property
    def ptrs(self) -> list:
        if self._list is None:
            self._list = [int(v) for v in self._np]
        return self._list


def _fresh(engine: CkksEngine, cem: ColumnEncodedMatrix) -> ColumnEncodedMatrix:
    """Operand fresh from one encryption batch: same engine, top level, depth 0 for every
    ciphertext, so the validated pointer cache of _checked_ptrs can be filled directly -- from the
    batch's base address and stride, without creating the Ciphertext objects."""
    cts = cem.cts
    if isinstance(cts, CtBatch):
        cache = _OperandCache(engine._id, engine.L, 0, _Storages([cts.out]), np_ptrs=cts.pointers())
    else:
        cache = _OperandCache(engine._id, engine.L, 0, _storages(cts), ptrs=[c._ptr for c in cts])
    object.__setattr__(cem, "_vr_ptrs", cache)
    return cem


class _Storages(list):
    """The distinct device tensors behind a list of ciphertexts (batches share one), plus the slot
    streams they were already recorded on: the caching allocator keeps a recorded stream for the
    block's lifetime, so each (tensor, stream) pair is recorded once, not per product."""

    __slots__ = ("recorded",)

    def record(self, stream, key: int) -> None:
        rec = getattr(self, "recorded", None)
        if rec is None:
            rec = self.recorded = set()
        if key not in rec:
            for t in self:
                t.record_stream(stream)
            rec.add(key)


def _storages(cts):
    if isinstance(cts, CtBatch):
        return _Storages([cts.out])
    seen = {}
    for c in cts:
        t = c.storage_tensor()
        seen.setdefault(id(t), t)
    return _Storages(seen.values())


def _layout0(cts):
    """Layout tag of the first ciphertext (without materialising a lazy batch)."""
    return cts.layout if isinstance(cts, CtBatch) else cts[0].layout


def _common_level(engine: CkksEngine, cts):
    lv = min(ct.level for ct in cts)
    if all(ct.level == lv for ct in cts):
        return cts, lv
    return [engine.adjust(ct, lv) for ct in cts], lv


def _checked_ptrs(engine: CkksEngine, cem: ColumnEncodedMatrix):
    """(level, [device pointers]) of a column-encoded operand, validated and cached on the object
    (operands are immutable; the cache also holds the ctypes pointer array and the max depth)."""
    cached = getattr(cem, "_vr_ptrs", None)
    if cached is not None and cached.eid == engine._id:
        return cached.level, cached.ptrs
    for c in cem.cts:
        engine._check(c)
    lv = min(c.level for c in cem.cts)
    ptrs = None
    if all(c.level == lv for c in cem.cts):
        ptrs = [c.ptr() for c in cem.cts]
        object.__setattr__(cem, "_vr_ptrs", _OperandCache(engine._id, lv, max(c.depth for c in cem.cts), _storages(cem.cts),
                                                          ptrs=ptrs))
    return lv, ptrs


def _fast_operand(engine: CkksEngine, cem: ColumnEncodedMatrix):
    """The operand's validated cache (level, arr, depth, storages) for this engine, or None."""
    cached = getattr(cem, "_vr_ptrs", None)
    if cached is not None and cached.eid == engine._id:
        return cached
    return None


def matmul_outer(engine: CkksEngine, left: ColumnEncodedMatrix, right: ColumnEncodedMatrix) -> PackedMatrix:
    """Sum of the n slot-wise products; no rotations, depth + 1 (multicipher.py:88-103)."""
    if left.role != "left" or right.role != "right":
        raise LayoutError("operands must be a (left, right) column-encoded pair")
    if (left.n, left.m, left.p) != (right.n, right.m, right.p):
        raise LayoutError(
            f"operand dims differ: left {(left.m, left.n, left.p)}, right {(right.m, right.n, right.p)}"
        )
    ct = matmul_outer_blocks(engine, [left], right)[0]
    return PackedMatrix(ct, MatrixShape(left.m, left.p), Encoding.ROW_MAJOR)


def matmul_outer_blocks(engine: CkksEngine, lefts, right: ColumnEncodedMatrix) -> list[Ciphertext]:
    """Row-tiled matmul_outer: block b = sum_k L_b,k * R_k for 1, 2 or 4 blocks sharing R.

    Meter: per block exactly the reference's n muls and n-1 adds.
    """
    nb = len(lefts)
    if nb not in (1, 2, 4):
        raise EngineError("matmul_outer_blocks supports 1, 2 or 4 row blocks")
    n = right.n
    if nb == 1:
        # steady state (operands already validated once): cached pointer arrays, no per-call scans
        fl, fr = _fast_operand(engine, lefts[0]), _fast_operand(engine, right)
        lf = lefts[0]
        if (fl is not None and fr is not None and fl.level == fr.level and fl.level >= 1 and lf.role == "left"
                and right.role == "right" and lf.n == n and lf.p == right.p):
            lv = fl.level
            pending = None
            if engine.async_drivers:
                # asynchronous: the product runs on a library slot stream, overlapping the next calls.
                # The output is allocated ON that stream (the caching allocator then reuses it in that
                # stream's order, with no cross-stream events), the operands are recorded on it once,
                # and any read of the result waits for it (Ciphertext._ready)
                engine._adopt_stream()
                h = engine._h
                slot = ctypes.c_void_p()
                _lib.check(engine._lib.vr_async_slot(h, ctypes.byref(slot)))
                ext = engine._ext_stream(slot.value)
                if engine._enc_queue:  # the operands' deferred encryption runs on the product's slot stream
                    engine._flush_enc(on=ext if engine._enc_on_slot else None)
                for op in (lf.cts, right.cts):  # operands produced on another side stream
                    if type(op) is CtBatch and op._pending is not None:
                        op.order_on(ext)
                outs = engine._empty_on(ext, (1, 2, lv, engine.N))
                _lib.check(engine._lib.vr_matmul_outer_async(h, fl.arr, fr.arr, n, 1, lv, _lib.row_ptrs(outs, 1),
                                                             ctypes.byref(slot)))
                if slot.value:
                    pending = ext
                    fl.storages.record(pending, slot.value)
                    fr.storages.record(pending, slot.value)
                else:  # ran synchronously on the current stream
                    outs.record_stream(torch.cuda.current_stream(engine.device))
            else:
                outs = torch.empty((1, 2, lv, engine.N), dtype=torch.int64, device=engine.device)
                _lib.check(engine._lib.vr_matmul_outer(engine.handle, fl.arr, fr.arr, n, 1, lv, _lib.row_ptrs(outs, 1)))
            depth = max(fl.depth, fr.depth) + 1
            engine._meter.mul_count += n
            engine._meter.add_count += n - 1
            engine._observe(depth)
            ct = Ciphertext.at(outs, 0, lv - 1, engine.scales[lv - 1], depth, _layout0(lf.cts), engine._id)
            ct._pending = pending
            return [ct]
    for lf in lefts:
        if lf.role != "left" or right.role != "right":
            raise LayoutError("operands must be a (left, right) column-encoded pair")
        if lf.n != n or lf.p != right.p:
            raise LayoutError("row blocks must share n and p with the right operand")
    infos = [_checked_ptrs(engine, lf) for lf in lefts] + [_checked_ptrs(engine, right)]
    lvs = {lv for lv, _ in infos}
    if len(lvs) == 1 and all(p is not None for _, p in infos):
        lv = lvs.pop()
        lptrs = [p for _, ps in infos[:-1] for p in ps]
        rptrs = infos[-1][1]
    else:
        allc, lv = _common_level(engine, [c for lf in lefts for c in lf.cts] + list(right.cts))
        lptrs = [c.ptr() for c in allc[: nb * n]]
        rptrs = [c.ptr() for c in allc[nb * n:]]
    if lv < 1:
        raise EngineError("multiplicative depth exhausted: operands are at level 0")
    outs = torch.empty((nb, 2, lv, engine.N), dtype=torch.int64, device=engine.device)
    _lib.check(engine._lib.vr_matmul_outer(
        engine.handle, _lib.ptr_array(lptrs), _lib.ptr_array(rptrs), n, nb, lv,
        _lib.row_ptrs(outs, nb)))
    rdepth = max(c.depth for c in right.cts)
    res = []
    for b, lf in enumerate(lefts):
        depth = max(rdepth, max(c.depth for c in lf.cts)) + 1
        engine._meter.mul_count += n
        engine._meter.add_count += n - 1
        engine._observe(depth)
        res.append(Ciphertext.at(outs, b, lv - 1, engine.scales[lv - 1], depth, _layout0(lf.cts), engine._id))
    return res


def matmul_outer_many(engine: CkksEngine, pairs) -> list[PackedMatrix]:
    """``[matmul_outer(engine, l, r) for l, r in pairs]`` as one launch sequence (vr_matmul_outer_many).

    Every pair must have the same n (column ciphertexts per operand) and all operands the same level.
    Small products are bound by kernel launches, not bytes: the batch shares one tensor-sum launch and
    one relinearise + rescale chain.  Residues, meter counts and depths are those of separate calls
    (multicipher.py:88-103 once per pair).
    """
    pairs = list(pairs)
    if not pairs:
        return []
    n = pairs[0][1].n
    for left, right in pairs:
        if left.role != "left" or right.role != "right":
            raise LayoutError("operands must be a (left, right) column-encoded pair")
        if (left.n, left.m, left.p) != (right.n, right.m, right.p):
            raise LayoutError(
                f"operand dims differ: left {(left.m, left.n, left.p)}, right {(right.m, right.n, right.p)}"
            )
        if left.n != n:
            raise LayoutError("matmul_outer_many needs the same n for every pair")
    caches = []
    for left, right in pairs:  # validated once per operand, then served from the operand's cache
        for cem in (left, right):
            c = _fast_operand(engine, cem)
            if c is None:
                _checked_ptrs(engine, cem)
                c = _fast_operand(engine, cem)
                if c is None:
                    raise LayoutError("matmul_outer_many needs every operand ciphertext at one common level")
            caches.append(c)
    lv = caches[0].level
    if any(c.level != lv for c in caches):
        raise LayoutError("matmul_outer_many needs every operand ciphertext at one common level")
    if lv < 1:
        raise EngineError("multiplicative depth exhausted: operands are at level 0")
    cnt = len(pairs)
    lnp = np.concatenate([c._np for c in caches[0::2]])
    rnp = np.concatenate([c._np for c in caches[1::2]])
    h = engine.handle  # adopts the current stream and launches deferred encryptions
    outs = torch.empty((cnt, 2, lv, engine.N), dtype=torch.int64, device=engine.device)
    onp = outs.data_ptr() + np.arange(cnt, dtype=np.uint64) * np.uint64(outs.stride(0) * 8)
    as_arr = lambda a: (ctypes.c_void_p * a.size).from_buffer(a)  # noqa: E731
    _lib.check(engine._lib.vr_matmul_outer_many(h, as_arr(lnp), as_arr(rnp), n, cnt, lv, as_arr(onp)))
    engine._meter.mul_count += n * cnt
    engine._meter.add_count += (n - 1) * cnt
    res = []
    level, scale = lv - 1, engine.scales[lv - 1]
    for b, (left, right) in enumerate(pairs):
        depth = max(caches[2 * b].depth, caches[2 * b + 1].depth) + 1
        engine._observe(depth)
        ct = Ciphertext.at(outs, b, level, scale, depth, _layout0(left.cts), engine._id)
        res.append(PackedMatrix(ct, MatrixShape(left.m, left.p), Encoding.ROW_MAJOR))
    return res


def encode_image_columns(engine: CkksEngine, images) -> ColumnEncodedImage:
    """Split images into per-column ciphertexts (batch at stride h), multicipher.py:106-120."""
    arr = np.asarray(images, dtype=np.float64)
    if arr.ndim == 2:
        arr = arr[None, :, :]
    if arr.ndim != 3:
        raise EngineError(f"expected one image or a batch, got ndim={arr.ndim}")
    m, h, w = arr.shape
    if m * h > engine.slots:
        raise CapacityError(f"{m} columns of {h} pixels need {m * h} slots")
    # column j: slot b*h + i = img[b, i, j], gathered on the device from the raw images
    cts = engine.enc_strided(arr, count=w, nvals=m * h, p=h, sc=1, s1=h * w, s2=w, layout=("column", h, m))
    return ColumnEncodedImage(cts, h, w, m, stride=h)


def pad_images(images, pad: int) -> np.ndarray:
    """Zero padding on the host (the reference conv is valid-only, multicipher.py:132-134)."""
    arr = np.asarray(images, dtype=np.float64)
    widths = [(0, 0)] * (arr.ndim - 2) + [(pad, pad), (pad, pad)]
    return np.pad(arr, widths)


def conv_constants(engine: CkksEngine, level: int, scale: float, weights, biases):
    """Integer tap weights, bias residues and the mask scale for the fused conv.

    acc = sum w_int * x has scale ``scale * 2^delta_c``; the valid mask is encoded at
    s_m = s[level] / 2^delta_c so that mask * acc, rescaled by q[level], lands exactly
    on the canonical s[level-1].
    """
    dc = float(2 ** engine.params.delta_c)
    w = np.asarray(weights, dtype=np.float64)
    w_int = np.array([int(round(float(x) * dc)) for x in w.reshape(-1)], dtype=np.int64).reshape(w.shape)
    # the bias integer lives at scale * 2^delta_c and can exceed 64 bits: pass exact residues
    b_ints = [int(round(float(b) * scale * dc)) for b in np.asarray(biases, dtype=np.float64).reshape(-1)]
    b_res = np.array([[bi % engine.q[i] for i in range(level + 1)] for bi in b_ints], dtype=np.uint64)
    mask_scale = engine.scales[level] / dc
    return w_int, b_res, mask_scale


def _valid_mask(m: int, stride: int, out_h: int) -> np.ndarray:
    valid = np.zeros((m, stride), dtype=np.float64)
    valid[:, :out_h] = 1.0
    return valid.reshape(-1)


def conv_columns(engine: CkksEngine, img: ColumnEncodedImage, kernel: Kernel) -> ColumnEncodedImage:
    """Valid convolution in the column domain (multicipher.py:123-162)."""
    k = kernel.k
    if k > img.h or k > img.w:
        raise EngineError(f"{k}x{k} kernel larger than {img.h}x{img.w} image")
    w4 = kernel.weights[None, None, :, :]
    return conv_columns_multi(engine, [img], w4, [kernel.bias])[0]


def _meter_conv_call(engine: CkksEngine, weights2d: np.ndarray, out_cols, depth_in: int) -> None:
    """Meter exactly what one reference conv_columns call records (multicipher.py:139-161)."""
    k = weights2d.shape[0]
    nz = [(p, q) for q in range(k) for p in range(k) if weights2d[p, q] != 0.0]
    rots = {(jp + q, p) for jp in out_cols for (p, q) in nz if p != 0}
    m = engine._meter
    m.rot_count += len(rots)
    m.enc_count += len(out_cols)
    m.cmul_count += len(nz) * len(out_cols)
    m.add_count += len(nz) * len(out_cols)
    engine._observe(depth_in + (1 if nz else 0))


def conv_columns_multi(engine: CkksEngine, imgs, weights, biases, out_cols=None) -> list[ColumnEncodedImage]:
    """F-filter, C-channel column convolution in one driver call.

    ``weights`` is [F][C][k][k]; output filter f = sum_c conv_columns(imgs[c], K[f][c]) + bias[f],
    restricted to ``out_cols`` (default: every valid column).  Rotations are computed once per
    (channel, column, shift) and shared by all filters; the meter records the reference
    composition (one conv_columns per (f, c) plus C-1 channel adds per filter).
    """
    imgs = list(imgs)
    w = np.asarray(weights, dtype=np.float64)
    if w.ndim != 4 or w.shape[2] != w.shape[3]:
        raise EngineError(f"weights must be [F][C][k][k], got {w.shape}")
    F, C, k, _ = w.shape
    if len(imgs) != C:
        raise LayoutError(f"{C} weight channels but {len(imgs)} images")
    base = imgs[0]
    for im in imgs:
        if (im.h, im.w, im.m, im.stride) != (base.h, base.w, base.m, base.stride):
            raise LayoutError("channel images must share h, w, m and stride")
    if k > base.h or k > base.w:
        raise EngineError(f"{k}x{k} kernel larger than {base.h}x{base.w} image")
    out_h, out_w = base.h - k + 1, base.w - k + 1
    cols = list(range(out_w)) if out_cols is None else [int(c) for c in out_cols]
    if any(c < 0 or c >= out_w for c in cols):
        raise EngineError("output column out of range")
    biases = np.broadcast_to(np.asarray(biases, dtype=np.float64).reshape(-1), (F,))
    X = [ct for im in imgs for ct in im.cts]
    for ct in X:
        engine._check(ct)
    X, lv = _common_level(engine, X)
    if lv < 1:
        raise EngineError("multiplicative depth exhausted: operands are at level 0")
    w_int, b_int, mask_scale = conv_constants(engine, lv, X[0].scale, w, biases)
    mask_pt = engine.encode_plain(_valid_mask(base.m, base.stride, out_h), lv, mask_scale)
    nout = len(cols)
    Y = torch.empty((F, nout, 2, lv, engine.N), dtype=torch.int64, device=engine.device)
    yptrs = [Y[f, o].data_ptr() for f in range(F) for o in range(nout)]
    w_c = np.ascontiguousarray(w_int, dtype=np.int64)
    b_c = np.ascontiguousarray(b_int, dtype=np.uint64)
    cols_c = (ctypes.c_int * max(1, nout))(*cols)
    _lib.check(engine._lib.vr_conv_columns(
        engine.handle, _lib.ptr_array([c.ptr() for c in X]), C, base.w, k,
        w_c.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), b_c.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), F,
        cols_c, nout, mask_pt.data_ptr(), lv, _lib.ptr_array(yptrs)))
    depth_in = max(ct.depth for ct in X)
    out = []
    for f in range(F):
        for c in range(C):
            _meter_conv_call(engine, w[f, c], cols, depth_in)
        engine._meter.add_count += C - 1
        cts = [Ciphertext.at(Y[f], o, lv - 1, engine.scales[lv - 1], depth_in + 1, ("column", out_h, base.m), engine._id)
               for o in range(nout)]
        out.append(ColumnEncodedImage(cts, out_h, nout, base.m, base.stride))
    return out


def reassemble_columns(engine: CkksEngine, img: ColumnEncodedImage) -> np.ndarray:
    """Decode to an (m, h, w) array (multicipher.py:165-172); one batched decrypt."""
    # only the slots the reference reads (b * stride + i, i < h) are copied to the host
    sel = (np.arange(img.m)[:, None] * img.stride + np.arange(img.h)[None, :]).reshape(-1)
    vecs = engine.dec_batch(img.cts, select=sel)  # [w][m * h]
    return np.ascontiguousarray(vecs.reshape(len(img.cts), img.m, img.h).transpose(1, 2, 0))
