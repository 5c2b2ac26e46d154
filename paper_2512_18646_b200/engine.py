"""CkksEngine: the reference SlotEngine surface (engine.py:167-251) backed by
RNS-CKKS on the B200 through libvrhe.so.

Same methods, signatures, meter semantics and exceptions as the simulator:
``enc, dec, add, mul, cmul, rot, mask, meter_snapshot, slots, params``.  A
ciphertext carries (device residues, level, scale, depth, layout); depth keeps
the reference's bookkeeping (add: max, mul/cmul: +1) and always equals
``L - level`` because every multiplication consumes exactly one prime.

Scale management: every level l has one canonical scale
s[l] (s[L] = 2^delta, s[l-1] = s[l]^2 / q[l]).  Products are rescaled
immediately, plaintext/constant operands are encoded at s[l], and an ``add``
of operands at different levels brings the higher one down with one integer
scalar multiplication + rescale, so results are always at the canonical scale
of their level.  All of this runs on the GPU; the host only does bookkeeping.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib
from .errors import CapacityError, EngineError, LayoutError
from .params import EngineParams, is_pow2, next_pow2

__all__ = [
    "EngineError",
    "CapacityError",
    "LayoutError",
    "EngineParams",
    "OpMeter",
    "Ciphertext",
    "PlainMask",
    "CkksEngine",
    "DecodeFuture",
    "SlotEngine",
    "is_pow2",
    "next_pow2",
]


@dataclass
class OpMeter:
    """Operation counters, identical to engine.py:93-131."""

    add_count: int = 0
    mul_count: int = 0
    cmul_count: int = 0
    rot_count: int = 0
    enc_count: int = 0
    max_depth: int = 0

    def copy(self) -> "OpMeter":
        return replace(self)

    def merged(self, other: "OpMeter") -> "OpMeter":
        return OpMeter(
            add_count=self.add_count + other.add_count,
            mul_count=self.mul_count + other.mul_count,
            cmul_count=self.cmul_count + other.cmul_count,
            rot_count=self.rot_count + other.rot_count,
            enc_count=self.enc_count + other.enc_count,
            max_depth=max(self.max_depth, other.max_depth),
        )

    def delta_since(self, earlier: "OpMeter") -> "OpMeter":
        return OpMeter(
            add_count=self.add_count - earlier.add_count,
            mul_count=self.mul_count - earlier.mul_count,
            cmul_count=self.cmul_count - earlier.cmul_count,
            rot_count=self.rot_count - earlier.rot_count,
            enc_count=self.enc_count - earlier.enc_count,
            max_depth=self.max_depth,
        )


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None) or (
    lambda dev: torch.cuda.current_stream(dev).cuda_stream)  # the current stream's cudaStream_t, cheaply


_cur_stream_raw = getattr(torch._C, "_cuda_getCurrentStream", None)  # (stream_id, device_index, device_type)
_set_stream_raw = getattr(torch._C, "_cuda_setStream", None)


def scalar_i64(x: float) -> int:
    """round(x) as a signed 64-bit scalar for the C-ABI; ctypes would wrap larger values silently."""
    k = int(round(x))
    if not -(1 << 63) < k < (1 << 63):
        raise CapacityError(f"constant {x:.6g} does not fit a 64-bit integer scalar at this scale")
    return k


def _frozen(values) -> np.ndarray:
    out = np.array(values, dtype=np.float64)
    out.flags.writeable = False
    return out


class _FailedProducer:
    """Pending marker of ciphertexts whose deferred encryption raised: every later use raises too
    instead of reading residues that were never written."""

    __slots__ = ("why",)

    def __init__(self, why: str):
        self.why = why


class Ciphertext:
    """RNS-CKKS ciphertext: residues [degree+1][level+1][N] on the GPU (treated as immutable).

    Ciphertexts produced by one batched kernel share its [count][degree+1][level+1][N] output;
    each keeps (batch, index) plus its device address and materialises the ``data`` view only
    when asked, so wrapping a 64-ciphertext batch costs no per-item tensor indexing.
    """

    __slots__ = ("_data", "_batch", "_idx", "_ptr", "level", "scale", "depth", "layout", "engine_id", "_pending")

    def __init__(self, data: torch.Tensor, level: int, scale: float, depth: int = 0, layout: tuple | None = None,
                 engine_id: int = 0):
        self._data = data
        self._batch = None
        self._idx = 0
        self._pending = None
        self._ptr = data.data_ptr()
        self.level = level
        self.scale = scale
        self.depth = depth
        self.layout = layout
        self.engine_id = engine_id

    @classmethod
    def at(cls, out: torch.Tensor, i: int, level: int, scale: float, depth: int = 0, layout: tuple | None = None,
           engine_id: int = 0) -> "Ciphertext":
        """Ciphertext ``out[i]`` of a contiguous batch, without creating the view."""
        ct = cls.__new__(cls)
        ct._data = None
        ct._batch = out
        ct._pending = None
        ct._idx = i
        ct._ptr = out.data_ptr() + i * out.stride(0) * out.element_size()
        ct.level = level
        ct.scale = scale
        ct.depth = depth
        ct.layout = layout
        ct.engine_id = engine_id
        return ct

    @classmethod
    def batch(cls, out: torch.Tensor, level: int, scale: float, depth: int = 0, layout: tuple | None = None,
              engine_id: int = 0, count: int | None = None) -> list["Ciphertext"]:
        """One ciphertext per leading index of ``out`` ([count][deg+1][l+1][N], contiguous)."""
        base, step = out.data_ptr(), out.stride(0) * out.element_size()
        res = []
        new = cls.__new__
        for i in range(out.shape[0] if count is None else count):
            ct = new(cls)
            ct._data = None
            ct._batch = out
            ct._pending = None
            ct._idx = i
            ct._ptr = base + i * step
            ct.level = level
            ct.scale = scale
            ct.depth = depth
            ct.layout = layout
            ct.engine_id = engine_id
            res.append(ct)
        return res

    def _ready(self) -> None:
        """Order the current stream after the (asynchronous) producer of these residues, and record
        the storage on the current stream: the producer's stream owns the allocation, so reads
        queued here must complete before the caching allocator hands the block out again."""
        p = self._pending
        if p is not None:
            if isinstance(p, _FailedProducer):
                raise EngineError(f"the deferred encryption of this ciphertext failed: {p.why}")
            if isinstance(p, CkksEngine):  # a deferred encryption: launch it (and its queue) now
                p._flush_enc()
                if self._pending is None or self._pending is p:
                    return
                return self._ready()  # launched on a side stream, or failed
            cur = torch.cuda.current_stream()
            cur.wait_stream(p)
            self.storage_tensor().record_stream(cur)
            self._pending = None

    @property
    def data(self) -> torch.Tensor:
        self._ready()
        if self._data is None:
            self._data = self._batch[self._idx]
        return self._data

    def storage_tensor(self) -> torch.Tensor:
        """The device tensor holding these residues (a batch may hold several ciphertexts)."""
        return self._data if self._data is not None else self._batch

    @property
    def degree(self) -> int:
        return (self._batch.shape[1] if self._data is None else self._data.shape[0]) - 1

    def ptr(self) -> int:
        self._ready()
        return self._ptr

    def residues(self) -> np.ndarray:
        """Copy of the residues as uint64 numpy (for parity checks)."""
        return self.data.cpu().numpy().view(np.uint64)


@dataclass(frozen=True, eq=False)
class PlainMask:
    """Plaintext constant vector for cmul (engine.py:153-164).  Filter masks are 0/1."""

    values: np.ndarray
    role: str = "constant"

    def __post_init__(self):
        if self.role == "filter":
            vals = self.values
            if not np.all((vals == 0.0) | (vals == 1.0)):
                raise EngineError("filter masks may contain only 0.0 and 1.0")


class DecodeFuture:
    """Result of ``CkksEngine.dec_batch_async``: ``result()`` waits for the copy and returns the
    decoded slots as numpy (``post`` applied)."""

    __slots__ = ("_done", "_host", "_post")

    def __init__(self, done, host, post=None):
        self._done, self._host, self._post = done, host, post

    def result(self) -> np.ndarray:
        self._done.synchronize()
        out = self._host.numpy()
        return self._post(out) if self._post is not None else out


class TicketFuture:
    """Result of ``dec_batch_async`` on the library's own decode tickets (``vr_decode_submit``): the
    decrypt + decode + copy into a pinned buffer owned by the context are queued by ONE C call;
    ``result()`` waits for the ticket's event and returns the slots as a fresh numpy array."""

    __slots__ = ("_engine", "_ticket", "_shape", "_post", "_out")

    def __init__(self, engine, ticket, shape, post=None):
        self._engine, self._ticket, self._shape, self._post, self._out = engine, ticket, shape, post, None

    def result(self) -> np.ndarray:
        if self._out is None:
            out = np.empty(self._shape, dtype=np.float64)
            eng = self._engine
            if not eng._h:
                raise EngineError("the engine of this decode future has been destroyed")
            _lib.check(eng._lib.vr_decode_wait(eng._h, self._ticket, out.ctypes.data))
            self._ticket = -1
            self._out = self._post(out) if self._post is not None else out
        return self._out

    def __del__(self):
        t = getattr(self, "_ticket", -1)
        if t is not None and t >= 0 and getattr(self._engine, "_h", None):
            try:  # an abandoned future still has to hand its ticket back
                self._engine._lib.vr_decode_wait(self._engine._h, t, None)
            except Exception:
                pass


class CtBatch:
    """The ciphertexts of one batched kernel output ([count][deg+1][l+1][N]) as a list-like
    sequence whose ``Ciphertext`` objects are created on first access: an operand that only feeds
    ``matmul_outer`` never materialises them (its pointer table is base + i * stride)."""

    __slots__ = ("out", "level", "scale", "depth", "layout", "engine_id", "count", "_items", "_pending", "_evt")

    def __init__(self, out, level, scale, depth, layout, engine_id, count=None, pending=None):
        self.out, self.level, self.scale, self.depth = out, level, scale, depth
        self.layout, self.engine_id = layout, engine_id
        self.count = out.shape[0] if count is None else count
        self._items = None
        self._pending = pending  # the engine (encryption deferred) or the stream that produced the residues
        self._evt = None         # completion event of that producer, when it ran on a side stream

    def _all(self) -> list:
        items = self._items
        if items is None:
            items = self._items = Ciphertext.batch(self.out, self.level, self.scale, self.depth, self.layout,
                                                   self.engine_id, self.count)
            if self._pending is not None:
                for ct in items:
                    ct._pending = self._pending
        return items

    def set_pending(self, owner, new=None, evt=None) -> None:
        """The producer ``owner`` of this batch is done or has been launched: ``new`` is None (ordered on
        the current stream) or the side stream it runs on (readers on other streams wait for it)."""
        if self._pending is owner:
            self._pending = new
            self._evt = evt
            if self._items is not None:
                for ct in self._items:
                    if ct._pending is owner:
                        ct._pending = new

    def order_on(self, stream) -> None:
        """Make ``stream`` see these residues: nothing to do when it produced them or they are complete."""
        pend = self._pending
        if pend is None or pend is stream:
            return
        if isinstance(pend, _FailedProducer):
            raise EngineError(f"the deferred encryption of these ciphertexts failed: {pend.why}")
        evt = self._evt
        if evt is None:
            stream.wait_stream(pend)
        elif evt.query():  # the producer finished: settled for every stream
            self.set_pending(pend, None)
        else:
            stream.wait_event(evt)

    def pointers(self) -> np.ndarray:
        """Device addresses of the ciphertexts (uint64), without creating them."""
        step = self.out.stride(0) * self.out.element_size()
        return self.out.data_ptr() + step * np.arange(self.count, dtype=np.uint64)

    def __len__(self) -> int:
        return self.count

    def __getitem__(self, i):
        return self._all()[i]

    def __iter__(self):
        return iter(self._all())

    def __add__(self, other):
        return self._all() + list(other)

    def __radd__(self, other):
        return list(other) + self._all()

    def __repr__(self) -> str:
        return f"CtBatch(count={self.count}, level={self.level})"


class CkksEngine:
    """Metered RNS-CKKS engine over ``params.slots`` slots on one CUDA device."""

    def __init__(self, params: EngineParams | None = None, device: int | None = None):
        self.params = params if params is not None else EngineParams()
        if not torch.cuda.is_available():
            raise EngineError("CkksEngine needs a CUDA device (libvrhe has no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self._lib = _lib.load()
        p = self.params
        primes = (ctypes.c_uint64 * len(p.primes))(*p.primes)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self._lib.vr_ctx_create(p.log_n, len(p.prime_bits), primes, p.seed,
                                               1 if p.encryption == "secret" else 0, self.device.index,
                                               ctypes.byref(h)))
            self._stream = torch.cuda.current_stream(self.device)
        self._h = h
        self._stream_ptr = self._stream.cuda_stream
        self._dev_index = self.device.index
        _lib.check(self._lib.vr_set_stream(self._h, ctypes.c_void_p(self._stream_ptr)))
        self._meter = OpMeter()
        # asynchronous drivers (vr_matmul_outer_async): results are produced on the library's slot
        # streams and every read of them waits first (Ciphertext._ready); VR_ASYNC=0 disables
        self.async_drivers = os.environ.get("VR_ASYNC", "1") != "0"
        # deferred strided encryptions (secret-key engines): VR_DEFER_ENC=0 launches each at once
        self._defer_enc = p.encryption == "secret" and os.environ.get("VR_DEFER_ENC", "1") != "0"
        self._enc_queue = []
        # dec_batch_async through the library's decode tickets (one C call); VR_DECODE_TICKETS=0 keeps
        # the torch path (device tensor + pinned tensor + copy + event)
        self._decode_tickets = os.environ.get("VR_DECODE_TICKETS", "1") != "0"
        # VR_ENC_ON_SLOT=1: deferred operand encryptions run on the slot stream of the product that
        # consumes them, so the encryption of product i+1 overlaps the kernels of product i.  Measured
        # slower (e2e 4.3k -> 3.8k HE matmul/s: the 1024-CTA slot FFT and the 5120-CTA encryption NTT of
        # different products displace each other's CTAs), so off by default
        self._enc_on_slot = os.environ.get("VR_ENC_ON_SLOT", "0") == "1"
        self._ext_streams = {}
        self._nonce = 0
        self._pin = None
        self._pin_evt = None
        self.h2d_bytes = 0
        self.L = p.levels
        self.N = p.n
        self.q = list(p.primes)
        self.scales = p.scale_chain()
        self._id = id(self)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                self._lib.vr_ctx_destroy(h)
            except Exception:
                pass
            self._h = None

    # -- basics -----------------------------------------------------------
    @property
    def slots(self) -> int:
        return self.params.slots

    @property
    def handle(self):
        """The C context, ordered on the caller's CURRENT torch stream.

        Like a torch op, every engine call runs on ``torch.cuda.current_stream()``: the library
        kernels, the output allocations, the pinned H2D staging copies and the decode's D2H all
        share that one stream, so no cross-stream hazard exists inside a call.
        """
        self._adopt_stream()
        if self._enc_queue:
            self._flush_enc()
        return self._h

    def _adopt_stream(self) -> None:
        if _raw_stream(self._dev_index) != self._stream_ptr:
            cur = torch.cuda.current_stream(self.device)
            _lib.check(self._lib.vr_set_stream(self._h, ctypes.c_void_p(cur.cuda_stream)))
            self._stream, self._stream_ptr = cur, cur.cuda_stream

    def _observe(self, depth: int) -> None:
        if depth > self._meter.max_depth:
            self._meter.max_depth = depth

    def meter_snapshot(self) -> OpMeter:
        return self._meter.copy()

    def _empty(self, degree: int, level: int, count: int | None = None) -> torch.Tensor:
        shape = (degree + 1, level + 1, self.N) if count is None else (count, degree + 1, level + 1, self.N)
        return torch.empty(shape, dtype=torch.int64, device=self.device)

    def _wrap(self, data, level, depth, layout) -> Ciphertext:
        return Ciphertext(data, level, self.scales[level], depth, layout, self._id)

    def _check(self, ct: Ciphertext) -> None:
        if not isinstance(ct, Ciphertext) or ct.engine_id != self._id:
            raise EngineError("operands come from engines with different slot counts")

    def _check_pair(self, a: Ciphertext, b: Ciphertext) -> None:
        self._check(a)
        self._check(b)

    _PIN_RING = 8

    def _h2d(self, vals: np.ndarray) -> torch.Tensor:
        """Host float64 array -> device, staged through a ring of reusable pinned buffers: a buffer is
        refilled only after its previous copy has executed, so the host may run up to eight uploads
        ahead of the device (pipelined encrypt -> product -> decode steps)."""
        self._adopt_stream()  # the caller's current stream (no flush: an upload is not an engine call)
        nbytes = vals.nbytes
        if self._pin is None:
            self._pin = [None] * self._PIN_RING
            self._pin_evt = [None] * self._PIN_RING
            self._pin_next = 0
        i = self._pin_next
        self._pin_next = (i + 1) % self._PIN_RING
        if self._pin_evt[i] is not None:
            self._pin_evt[i].synchronize()
        if self._pin[i] is None or self._pin[i].numel() < vals.size:
            self._pin[i] = torch.empty(max(vals.size, 1 << 16), dtype=torch.float64, pin_memory=True)
        stage = self._pin[i][: vals.size].view(vals.shape)
        stage.numpy()[...] = vals
        out = torch.empty(vals.shape, dtype=torch.float64, device=self.device)
        out.copy_(stage, non_blocking=True)
        evt = self._pin_evt[i]
        if evt is None:
            evt = self._pin_evt[i] = torch.cuda.Event()
        evt.record(self._stream)
        self.h2d_bytes += nbytes
        return out

    def _pad(self, rows) -> np.ndarray:
        """List of value vectors -> zero-padded [count][width] float64 (width <= slots)."""
        vecs = [np.asarray(v, dtype=np.float64).reshape(-1) for v in rows]
        width = max([v.size for v in vecs] + [1])
        if width > self.slots:
            raise CapacityError(f"{width} values exceed {self.slots} slots")
        out = np.zeros((len(vecs), width), dtype=np.float64)
        for i, v in enumerate(vecs):
            out[i, : v.size] = v
        return out

    # -- primitive API (engine.py:193-251) ---------------------------------
    def enc(self, values, layout: tuple | None = None) -> Ciphertext:
        """Encode into the leading slots (zeros elsewhere) and encrypt at the top level."""
        return self.enc_batch([values], layout)[0]

    def enc_batch(self, rows, layout: tuple | None = None, nonce0: int | None = None) -> list[Ciphertext]:
        """``enc`` of many vectors in one launch (one enc_count each).

        Ciphertext i uses encryption nonce ``nonce0 + i`` (default: the engine's running
        counter).  An explicit ``nonce0`` lets sharded ranks reproduce exactly the
        ciphertexts a single-GPU run would have produced.
        """
        vals = self._pad(rows)
        count = vals.shape[0]
        d_vals = self._h2d(vals)
        out = self._empty(1, self.L, count)
        n0 = self._nonce if nonce0 is None else int(nonce0)
        _lib.check(self._lib.vr_encrypt(self.handle, d_vals.data_ptr(), count, vals.shape[1], self.L,
                                        self.scales[self.L], n0, out.data_ptr()))
        if nonce0 is None:
            self._nonce += count
        self._meter.enc_count += count
        self._observe(0)
        return Ciphertext.batch(out, self.L, self.scales[self.L], 0, layout, self._id)

    def enc_strided(self, src, count: int, nvals: int, p: int, sc: int, s1: int, s2: int, offset: int = 0,
                    layout: tuple | None = None, nonce0: int | None = None) -> list[Ciphertext]:
        """Encrypt ``count`` slot vectors gathered on the device from one raw host array.

        Ciphertext c holds slot j = src.flat[offset + c*sc + (j // p)*s1 + (j % p)*s2] for j < nvals
        (zeros beyond): the broadcast/tiling of encode_left/encode_right/encode_image_columns is done by
        the encode kernel, so only the raw matrix or images cross PCIe.
        """
        if nvals > self.slots:
            raise CapacityError(f"{nvals} values exceed {self.slots} slots")
        arr = np.ascontiguousarray(np.asarray(src, dtype=np.float64)).reshape(-1)
        defer = self._defer_enc and count > 0
        out = self._empty(1, self.L, count)
        n0 = self._nonce if nonce0 is None else int(nonce0)
        if defer and 0 < arr.nbytes <= self._HOST_STAGE_MAX:
            # small raw arrays stay on the host until the launch: the library stages them through its
            # pinned ring itself (vr_encrypt_strided*_host), one C call for copy + encode + encrypt.
            # The snapshot lets the caller reuse its array before the deferred launch.
            snap = arr.copy()
            job = (None, snap.ctypes.data, sc, s1, s2, max(1, p), nvals, count, n0, out, None, snap, int(offset))
            self.h2d_bytes += arr.nbytes
        else:
            d_src = self._h2d(arr) if arr.size else torch.zeros(1, dtype=torch.float64, device=self.device)
            job = (d_src, d_src.data_ptr() + 8 * int(offset), sc, s1, s2, max(1, p), nvals, count, n0, out, self._stream,
                   None, 0)
        if nonce0 is None:
            self._nonce += count
        self._meter.enc_count += count
        self._observe(0)
        cts = CtBatch(out, self.L, self.scales[self.L], 0, layout, self._id, count, self if defer else None)
        if defer:
            # deferred: launched at the next engine call or read of these ciphertexts (_flush_enc), so
            # the two operands of one product (encode_left + encode_right) become ONE encryption launch
            self._enc_queue.append((job, cts))
        else:
            self._launch_enc([job])
        return cts

    _HOST_STAGE_MAX = 1 << 20  # raw arrays up to 1 MB ride the library's pinned ring

    def _launch_enc(self, jobs) -> None:
        h = self._h
        L, scale = self.L, self.scales[self.L]
        if len(jobs) == 1:
            _, src, sc, s1, s2, p, nvals, count, n0, out, _, snap, off = jobs[0]
            if snap is not None:
                _lib.check(self._lib.vr_encrypt_strided_host(h, src, snap.size, off, sc, s1, s2, p, nvals, count, L, scale, n0,
                                                             out.data_ptr()))
            else:
                _lib.check(self._lib.vr_encrypt_strided(h, src, sc, s1, s2, p, nvals, count, L, scale, n0, out.data_ptr()))
            return
        ((_, a_src, a_sc, a_s1, a_s2, a_p, a_nv, a_cnt, a_n0, a_out, _, a_snap, a_off),
         (_, b_src, b_sc, b_s1, b_s2, b_p, b_nv, b_cnt, _, b_out, _, b_snap, b_off)) = jobs
        if a_snap is not None:
            _lib.check(self._lib.vr_encrypt_strided2_host(h, a_src, a_snap.size, a_off, a_sc, a_s1, a_s2, a_p, a_nv, a_cnt,
                                                          a_out.data_ptr(), b_src, b_snap.size, b_off, b_sc, b_s1, b_s2, b_p,
                                                          b_nv, b_cnt, b_out.data_ptr(), L, scale, a_n0))
        else:
            _lib.check(self._lib.vr_encrypt_strided2(h, a_src, a_sc, a_s1, a_s2, a_p, a_nv, a_cnt, a_out.data_ptr(), b_src, b_sc,
                                                     b_s1, b_s2, b_p, b_nv, b_cnt, b_out.data_ptr(), L, scale, a_n0))

    def _flush_enc(self, on=None) -> None:
        """Launch the deferred encryptions (consecutive-nonce pairs as one combined launch), ordered on
        the current stream after the streams their host copies were queued on -- or, with ``on``, on that
        side stream (the slot stream of the product that consumes them: the encryption of the next
        product then overlaps this product's kernels instead of queueing behind them on one stream)."""
        queue, self._enc_queue = self._enc_queue, []
        if not queue:
            return
        self._adopt_stream()
        cur = self._stream
        for (job, _) in queue:
            if job[10] is not None and job[10].cuda_stream != cur.cuda_stream:
                cur.wait_stream(job[10])
        if on is not None and on.cuda_stream == cur.cuda_stream:
            on = None
        if on is not None:  # `on` waits for the current stream, the context moves to it
            _lib.check(self._lib.vr_fork_stream(self._h, ctypes.c_void_p(on.cuda_stream)))
        try:
            groups = self._launch_queue(queue)
        except BaseException as exc:
            failed = _FailedProducer(str(exc) or type(exc).__name__)
            for (_, cts) in queue:  # nothing of this queue may be read as if it had been encrypted
                cts.set_pending(self, failed)
            raise
        finally:
            if on is not None:
                _lib.check(self._lib.vr_set_stream(self._h, ctypes.c_void_p(self._stream_ptr)))
        evt = None
        if on is not None:
            evt = torch.cuda.Event()
            evt.record(on)
        for g in groups:
            g.set_pending(self, on, evt)

    def _launch_queue(self, queue) -> list:
        done = []
        i = 0
        while i < len(queue):
            job, cts = queue[i]
            nxt = queue[i + 1][0] if i + 1 < len(queue) else None
            # nonces continue and both sources live on the same side (host / device): one launch
            if nxt is not None and nxt[8] == job[8] + job[7] and (nxt[11] is None) == (job[11] is None):
                self._launch_enc([job, nxt])
                group = [cts, queue[i + 1][1]]
                i += 2
            else:
                self._launch_enc([job])
                group = [cts]
                i += 1
            done.extend(group)
        return done

    def dec(self, ct: Ciphertext) -> np.ndarray:
        """Full slot vector (real parts), like engine.py:204-206."""
        return self.dec_batch([ct])[0]

    def dec_batch(self, cts, select=None) -> np.ndarray:
        """Decrypt + decode many ciphertexts -> [count][slots] (real parts).  ``select`` (slot
        indices) keeps only those slots, gathered on the device before the copy to the host."""
        return self._dec_device(cts, select).cpu().numpy()

    def _dec_device(self, cts, select=None) -> torch.Tensor:
        cts = list(cts)
        for ct in cts:
            self._check(ct)
        count = len(cts)
        out = torch.empty((count, self.slots), dtype=torch.float64, device=self.device)
        degs = (ctypes.c_int * count)(*[ct.degree for ct in cts])
        lvls = (ctypes.c_int * count)(*[ct.level for ct in cts])
        scl = (ctypes.c_double * count)(*[ct.scale for ct in cts])
        ptrs = _lib.ptr_array([ct.ptr() for ct in cts])
        _lib.check(self._lib.vr_decrypt_decode(self.handle, ptrs, degs, lvls, scl, count, out.data_ptr(), None))
        if select is not None:
            idx = torch.as_tensor(np.asarray(select, dtype=np.int64), device=self.device)
            out = out.index_select(1, idx)
        return out

    def dec_batch_async(self, cts, select=None, post=None) -> "DecodeFuture":
        """``dec_batch`` without blocking the host: decrypt + decode + the copy into pinned host
        memory are queued (on the producer's slot stream when every ciphertext comes from the same
        asynchronous driver call, else on the current stream) and ``DecodeFuture.result()`` waits.
        Lets a caller keep several encrypt -> product -> decode steps in flight."""
        cts = list(cts)
        pend = cts[0]._pending if cts else None
        on_slot = isinstance(pend, torch.cuda.Stream) and all(c._pending is pend for c in cts)
        if select is None and cts and self._decode_tickets:
            # one C call: the library decodes on the producer's stream (the ciphertexts were allocated
            # and written there) or on the current one, into its own pinned ticket buffer
            h = self.handle  # adopts the current stream, launches deferred encryptions
            for ct in cts:
                self._check(ct)
            count = len(cts)
            stream_ptr = pend.cuda_stream if on_slot else None
            ptrs = _lib.ptr_array([ct._ptr if on_slot else ct.ptr() for ct in cts])
            degs = (ctypes.c_int * count)(*[ct.degree for ct in cts])
            lvls = (ctypes.c_int * count)(*[ct.level for ct in cts])
            scl = (ctypes.c_double * count)(*[ct.scale for ct in cts])
            ticket = ctypes.c_int(-1)
            _lib.check(self._lib.vr_decode_submit(h, ptrs, degs, lvls, scl, count, stream_ptr, ctypes.byref(ticket)))
            # (the storages need no keep-alive: they are read on the stream that owns their allocation,
            # or were recorded on the current stream by ct.ptr())
            return TicketFuture(self, ticket.value, (count, self.slots), post)
        if on_slot:
            stream = pend
        else:
            self.handle  # noqa: B018 -- deferred encryptions first
            stream = torch.cuda.current_stream(self.device)
        with torch.cuda.stream(stream):
            out = self._dec_device(cts, select)
            host = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
            host.copy_(out, non_blocking=True)
            done = torch.cuda.Event()
            done.record(stream)
        return DecodeFuture(done, host, post)

    def add(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        self._check_pair(a, b)
        a2, b2 = self._align(a, b)
        depth = max(a.depth, b.depth)
        out = self._binop(a2, b2, 0)
        self._meter.add_count += 1
        self._observe(depth)
        return self._wrap(out, a2.level, depth, a.layout)

    def sub(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        """Not in the reference surface; metered as an add."""
        self._check_pair(a, b)
        a2, b2 = self._align(a, b)
        depth = max(a.depth, b.depth)
        out = self._binop(a2, b2, 1)
        self._meter.add_count += 1
        self._observe(depth)
        return self._wrap(out, a2.level, depth, a.layout)

    def mul(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        self._check_pair(a, b)
        a2, b2 = self._align(a, b)
        lv = a2.level
        if lv < 1:
            raise EngineError("multiplicative depth exhausted: operands are at level 0")
        out = self._empty(1, lv - 1)
        _lib.check(self._lib.vr_mul(self.handle, _lib.ptr_array([a2.ptr()]), _lib.ptr_array([b2.ptr()]),
                                    _lib.ptr_array([out.data_ptr()]), 1, lv))
        depth = max(a.depth, b.depth) + 1
        self._meter.mul_count += 1
        self._observe(depth)
        return self._wrap(out, lv - 1, depth, a.layout)

    def cmul(self, mask: PlainMask, ct: Ciphertext) -> Ciphertext:
        if mask.values.size != self.slots:
            raise EngineError(f"mask length {mask.values.size} != slot count {self.slots}")
        self._check(ct)
        lv = ct.level
        if lv < 1:
            raise EngineError("multiplicative depth exhausted: operand is at level 0")
        vals = mask.values
        tmp = self._empty(ct.degree, lv)
        if np.all(vals == vals[0]):
            k = scalar_i64(float(vals[0]) * ct.scale)
            _lib.check(self._lib.vr_mul_scalar(self.handle, _lib.ptr_array([ct.ptr()]), k,
                                               _lib.ptr_array([tmp.data_ptr()]), 1, ct.degree, lv))
        else:
            pt = self.encode_plain(vals, lv, ct.scale)
            _lib.check(self._lib.vr_mul_plain(self.handle, _lib.ptr_array([ct.ptr()]), _lib.ptr_array([pt.data_ptr()]),
                                              _lib.ptr_array([tmp.data_ptr()]), 1, ct.degree, lv, 1))
        out = self._empty(ct.degree, lv - 1)
        _lib.check(self._lib.vr_rescale(self.handle, _lib.ptr_array([tmp.data_ptr()]), _lib.ptr_array([out.data_ptr()]),
                                        1, ct.degree, lv))
        depth = ct.depth + 1
        self._meter.cmul_count += 1
        self._observe(depth)
        return self._wrap(out, lv - 1, depth, ct.layout)

    def rot(self, ct: Ciphertext, l: int) -> Ciphertext:
        """Cyclic left rotation by ``l`` slots; negative ``l`` rotates right."""
        self._check(ct)
        self._meter.rot_count += 1
        self._observe(ct.depth)
        if int(l) % self.slots == 0:
            return self._wrap(ct.data, ct.level, ct.depth, ct.layout)
        return self._wrap(self.rotate_many(ct, [int(l)])[0], ct.level, ct.depth, ct.layout)

    def mask(self, values, role: str = "constant") -> PlainMask:
        vec = np.asarray(values, dtype=np.float64).reshape(-1)
        if vec.size > self.slots:
            raise CapacityError(f"mask payload {vec.size} exceeds {self.slots} slots")
        full = np.zeros(self.slots, dtype=np.float64)
        full[: vec.size] = vec
        return PlainMask(_frozen(full), role=role)

    # -- batched forms of the reference ops ----------------------------------
    # Each computes exactly what the per-op loop would (same kernels, same
    # residues, same meter increments and depths) in one launch per stage.
    def _same_level(self, cts) -> bool:
        lv, sc = cts[0].level, cts[0].scale
        return all(c.level == lv and c.scale == sc for c in cts)

    def mul_batch(self, xs, ys) -> list[Ciphertext]:
        """[mul(x, y) for x, y in zip(xs, ys)] (operands may repeat)."""
        xs, ys = list(xs), list(ys)
        if len(xs) != len(ys):
            raise EngineError("mul_batch needs equally many left and right operands")
        if not xs:
            return []
        if not self._same_level(xs + ys):
            return [self.mul(x, y) for x, y in zip(xs, ys)]
        for c in xs + ys:
            self._check(c)
        lv, count = xs[0].level, len(xs)
        if lv < 1:
            raise EngineError("multiplicative depth exhausted: operands are at level 0")
        out = self._empty(1, lv - 1, count)
        _lib.check(self._lib.vr_mul(self.handle, _lib.ptr_array([x.ptr() for x in xs]), _lib.ptr_array([y.ptr() for y in ys]),
                                    _lib.row_ptrs(out), count, lv))
        res = []
        for i, (x, y) in enumerate(zip(xs, ys)):
            depth = max(x.depth, y.depth) + 1
            self._meter.mul_count += 1
            self._observe(depth)
            res.append(Ciphertext.at(out, i, lv - 1, self.scales[lv - 1], depth, x.layout, self._id))
        return res

    def cmul_batch(self, masks, cts) -> list[Ciphertext]:
        """[cmul(mask_i, ct_i)]; ``masks`` is one PlainMask (shared) or one per ciphertext."""
        cts = list(cts)
        if not cts:
            return []
        shared = isinstance(masks, PlainMask)
        masks = [masks] * len(cts) if shared else list(masks)
        if len(masks) != len(cts):
            raise EngineError("cmul_batch needs one mask per ciphertext (or one shared mask)")
        if not self._same_level(cts) or len({c.degree for c in cts}) != 1:
            return [self.cmul(m, c) for m, c in zip(masks, cts)]
        uniform = [bool(np.all(m.values == m.values[0])) for m in masks]
        if any(uniform):
            # constant masks take cmul's scalar path; the rest go through one batch
            res = [self.cmul(m, c) if u else None for m, c, u in zip(masks, cts, uniform)]
            rest = [i for i, u in enumerate(uniform) if not u]
            if rest:
                sub = self.cmul_batch(masks[0] if shared else [masks[i] for i in rest], [cts[i] for i in rest])
                for i, r in zip(rest, sub):
                    res[i] = r
            return res
        for m in masks:
            if m.values.size != self.slots:
                raise EngineError(f"mask length {m.values.size} != slot count {self.slots}")
        for c in cts:
            self._check(c)
        lv, deg, count, scale = cts[0].level, cts[0].degree, len(cts), cts[0].scale
        if lv < 1:
            raise EngineError("multiplicative depth exhausted: operand is at level 0")
        rows = [masks[0].values] if shared else [m.values for m in masks]
        vals = np.stack(rows)
        d_vals = self._h2d(vals)
        pts = torch.empty((len(rows), lv + 1, self.N), dtype=torch.int64, device=self.device)
        _lib.check(self._lib.vr_encode(self.handle, d_vals.data_ptr(), len(rows), self.slots, lv, scale, pts.data_ptr()))
        tmp = self._empty(deg, lv, count)
        _lib.check(self._lib.vr_mul_plain(self.handle, _lib.ptr_array([c.ptr() for c in cts]), _lib.row_ptrs(pts),
                                          _lib.row_ptrs(tmp), count, deg, lv, 1 if shared else 0))
        out = self._empty(deg, lv - 1, count)
        _lib.check(self._lib.vr_rescale(self.handle, _lib.row_ptrs(tmp), _lib.row_ptrs(out), count, deg, lv))
        res = []
        for i, c in enumerate(cts):
            self._meter.cmul_count += 1
            self._observe(c.depth + 1)
            res.append(Ciphertext.at(out, i, lv - 1, self.scales[lv - 1], c.depth + 1, c.layout, self._id))
        return res

    def add_batch(self, xs, ys) -> list[Ciphertext]:
        """[add(x, y) for x, y in zip(xs, ys)]."""
        xs, ys = list(xs), list(ys)
        if len(xs) != len(ys):
            raise EngineError("add_batch needs equally many operands")
        if not xs:
            return []
        if not self._same_level(xs + ys) or len({c.degree for c in xs + ys}) != 1:
            return [self.add(x, y) for x, y in zip(xs, ys)]
        for c in xs + ys:
            self._check(c)
        lv, deg, count = xs[0].level, xs[0].degree, len(xs)
        out = self._empty(deg, lv, count)
        _lib.check(self._lib.vr_add(self.handle, _lib.ptr_array([x.ptr() for x in xs]), _lib.ptr_array([y.ptr() for y in ys]),
                                    _lib.row_ptrs(out), count, deg, lv, 0))
        res = []
        for i, (x, y) in enumerate(zip(xs, ys)):
            depth = max(x.depth, y.depth)
            self._meter.add_count += 1
            self._observe(depth)
            res.append(Ciphertext.at(out, i, lv, x.scale, depth, x.layout, self._id))
        return res

    def rot_batch(self, cts, steps) -> list[list[Ciphertext]]:
        """[[rot(ct, s) for s in steps] for ct in cts]: one hoisted ModUp per ciphertext."""
        cts, steps = list(cts), [int(s) for s in steps]
        if not cts or not steps:
            return [[] for _ in cts]
        if not self._same_level(cts) or any(c.degree != 1 for c in cts):
            return [[self.rot(c, s) for s in steps] for c in cts]
        for c in cts:
            self._check(c)
        lv, count = cts[0].level, len(cts)
        nr = len(steps)
        flat = torch.empty((count * nr, 2, lv + 1, self.N), dtype=torch.int64, device=self.device)
        st = (ctypes.c_int64 * nr)(*steps)
        _lib.check(self._lib.vr_rotate(self.handle, _lib.ptr_array([c.ptr() for c in cts]), _lib.row_ptrs(flat),
                                       count, lv, nr, st))
        res = []
        for i, c in enumerate(cts):
            self._meter.rot_count += len(steps)
            self._observe(c.depth)
            res.append([Ciphertext.at(flat, i * nr + r, lv, c.scale, c.depth, c.layout, self._id) for r in range(nr)])
        return res

    def sum_batch(self, acc: Ciphertext, cts) -> Ciphertext:
        """acc + cts[0] + cts[1] + ... (``len(cts)`` adds, like the sequential loop).

        Modular addition is exact, so a pairwise tree over the aligned operands gives the
        same residues as the left-to-right chain.
        """
        cts = list(cts)
        if not cts:
            return acc
        lv = min([acc.level] + [c.level for c in cts])
        terms = [self.adjust(c, lv) for c in cts]
        if not self._same_level(terms) or terms[0].scale != self.scales[lv]:
            out = acc
            for c in cts:
                out = self.add(out, c)
            return out
        base = self.adjust(acc, lv)
        depth = max([acc.depth] + [c.depth for c in cts])
        m = self._meter
        before = m.add_count
        while len(terms) > 1:
            half = len(terms) // 2
            paired = self.add_batch(terms[:half], terms[half:2 * half])
            terms = paired + terms[2 * half:]
        out = self.add(base, terms[0])
        m.add_count = before + len(cts)
        self._observe(depth)
        return Ciphertext(out.data, out.level, out.scale, depth, acc.layout, self._id)

    # -- device-level helpers (no metering) --------------------------------
    def encode_plain(self, values, level: int, scale: float) -> torch.Tensor:
        vals = self._pad([values])
        d_vals = self._h2d(vals)
        pt = torch.empty((level + 1, self.N), dtype=torch.int64, device=self.device)
        _lib.check(self._lib.vr_encode(self.handle, d_vals.data_ptr(), 1, vals.shape[1], level, scale, pt.data_ptr()))
        return pt

    def _binop(self, a: Ciphertext, b: Ciphertext, op: int) -> torch.Tensor:
        if a.degree != b.degree:
            raise EngineError("operand degrees differ")
        out = self._empty(a.degree, a.level)
        _lib.check(self._lib.vr_add(self.handle, _lib.ptr_array([a.ptr()]), _lib.ptr_array([b.ptr()]),
                                    _lib.ptr_array([out.data_ptr()]), 1, a.degree, a.level, op))
        return out

    def rotate_many(self, ct: Ciphertext, steps) -> list[torch.Tensor]:
        """Hoisted rotations of one ciphertext (one ModUp shared by all amounts)."""
        steps = [int(s) for s in steps]
        outs = [self._empty(1, ct.level) for _ in steps]
        st = (ctypes.c_int64 * len(steps))(*steps)
        _lib.check(self._lib.vr_rotate(self.handle, _lib.ptr_array([ct.ptr()]), _lib.ptr_array([o.data_ptr() for o in outs]),
                                       1, ct.level, len(steps), st))
        return outs

    def adjust(self, ct: Ciphertext, level: int) -> Ciphertext:
        """Bring ``ct`` down to ``level`` at that level's canonical scale (no metering).

        Drop to level+1, multiply by round(s[level] * q[level+1] / scale), rescale.
        """
        if level == ct.level:
            return ct
        if level > ct.level:
            raise EngineError("cannot raise a ciphertext's level")
        cur, lv = ct, ct.level
        if lv > level + 1:
            dropped = self._empty(cur.degree, level + 1)
            _lib.check(self._lib.vr_drop_level(self.handle, _lib.ptr_array([cur.ptr()]), _lib.ptr_array([dropped.data_ptr()]),
                                               1, cur.degree, lv, level + 1))
            cur = Ciphertext(dropped, level + 1, ct.scale, ct.depth, ct.layout, self._id)
        k = scalar_i64(self.scales[level] * float(self.q[level + 1]) / cur.scale)
        tmp = self._empty(cur.degree, level + 1)
        _lib.check(self._lib.vr_mul_scalar(self.handle, _lib.ptr_array([cur.ptr()]), k, _lib.ptr_array([tmp.data_ptr()]),
                                           1, cur.degree, level + 1))
        out = self._empty(cur.degree, level)
        _lib.check(self._lib.vr_rescale(self.handle, _lib.ptr_array([tmp.data_ptr()]), _lib.ptr_array([out.data_ptr()]),
                                        1, cur.degree, level + 1))
        return Ciphertext(out, level, self.scales[level], ct.depth, ct.layout, self._id)

    def _align(self, a: Ciphertext, b: Ciphertext):
        if a.level == b.level:
            if a.scale != b.scale:
                raise EngineError("operands at the same level carry different scales")
            return a, b
        lv = min(a.level, b.level)
        return self.adjust(a, lv), self.adjust(b, lv)

    def sync(self) -> None:
        self.join()
        _lib.check(self._lib.vr_sync(self.handle))

    def join(self) -> None:
        """Make the current stream wait for every asynchronous driver call issued so far."""
        _lib.check(self._lib.vr_join(self.handle))
        side = self._ext_streams.get("side")
        if side is not None:
            torch.cuda.current_stream(self.device).wait_stream(side)

    def _side_stream(self):
        """A second stream of this engine for asynchronous finishing work (dist._finish_async)."""
        s = self._ext_streams.get("side")
        if s is None:
            s = self._ext_streams["side"] = torch.cuda.Stream(device=self.device)
        return s

    def _empty_on(self, stream, shape) -> torch.Tensor:
        """``torch.empty(shape, int64)`` allocated on ``stream`` (the caching allocator then reuses the
        block in that stream's order).  Switches torch's current stream through the C bindings the
        ``torch.cuda.stream`` context manager wraps: the manager's Python layers cost ~8 us per
        product, more than the library call it brackets."""
        get, put = _cur_stream_raw, _set_stream_raw
        if get is None or put is None:
            with torch.cuda.stream(stream):
                return torch.empty(shape, dtype=torch.int64, device=self.device)
        prev = get(self._dev_index)
        put(stream_id=stream.stream_id, device_index=stream.device_index, device_type=stream.device_type)
        try:
            return torch.empty(shape, dtype=torch.int64, device=self.device)
        finally:
            put(stream_id=prev[0], device_index=prev[1], device_type=prev[2])

    def _ext_stream(self, ptr: int):
        s = self._ext_streams.get(ptr)
        if s is None:
            s = self._ext_streams[ptr] = torch.cuda.ExternalStream(ptr, device=self.device)
        return s


# The reference name: algorithm modules construct ``SlotEngine(EngineParams(...))``.
SlotEngine = CkksEngine
