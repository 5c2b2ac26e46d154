"""Multi-GPU sharding of the column-ciphertext path.

* HE matmul (config 5a): C = sum_k L_k * R_k is a sum over independent column
  ciphertexts (multicipher.py:100-102).  Rank g owns a contiguous
  k range, computes the degree-2 partial sum locally (one fused tensor-sum
  launch for every row block), the partials are summed in int64 (every
  residue is < 2^60, so up to 8 ranks cannot overflow) -- either one NCCL
  all-reduce (every rank finishes every block) or one reduce per row block to
  its owner rank (``matmul_outer_sharded_owned``: each rank relinearises only
  its own blocks) -- then reduced mod q, relinearised and rescaled once.
  Because the modular sum is exact and relinearisation happens after it, the
  result is bit-identical for 1, 2, 4 or 8 ranks.
* HE conv (config 5b): images are independent; groups of images shard across
  ranks with no collective at all.

Encryption nonces follow the single-GPU order (``matmul_nonce_plan``) so a
sharded run reproduces exactly the ciphertexts of an unsharded one.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .engine import Ciphertext, CkksEngine, EngineError, LayoutError
from .multicipher import ColumnEncodedMatrix, _checked_ptrs

__all__ = ["shard_range", "matmul_nonce_plan", "encode_operands_sharded", "allreduce_partials", "block_owner",
           "reduce_partials_to_owners", "matmul_partials", "matmul_finish", "matmul_outer_sharded",
           "matmul_outer_sharded_owned", "image_groups", "NativeComm"]


class NativeComm:
    """NCCL communicator owned by the engine's C context (vr_comm_*): the partial-product sum of
    config 5a runs inside libvrhe (uint64 NCCL sum + mod-q reduction on the device) instead of
    through torch.distributed.  torch.distributed (any backend) is only used, in ``from_group``, to
    hand the 128-byte NCCL unique id from rank 0 to the other ranks."""

    def __init__(self, engine: CkksEngine, uid: bytes, rank: int, world: int):
        import ctypes

        if len(uid) != 128:
            raise EngineError("an NCCL unique id has 128 bytes")
        self.engine, self.rank, self.world = engine, rank, world
        buf = ctypes.create_string_buffer(uid, 128)
        _lib.check(engine._lib.vr_comm_init(engine.handle, buf, rank, world))

    @staticmethod
    def unique_id(engine: CkksEngine) -> bytes:
        import ctypes

        buf = ctypes.create_string_buffer(128)
        _lib.check(engine._lib.vr_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def from_group(cls, engine: CkksEngine, group=None) -> "NativeComm":
        import torch.distributed as dist

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        obj = [cls.unique_id(engine) if rank == 0 else None]
        src = 0 if group is None else dist.get_global_rank(group, 0)
        dist.broadcast_object_list(obj, src=src, group=group)
        return cls(engine, obj[0], rank, world)

    def sum_partials(self, part: torch.Tensor, level: int, root: int = -1) -> None:
        """In-place sum of [polys][level+1][N] residues over ranks, reduced mod q (root < 0: every rank)."""
        if part.dtype != torch.int64 or not part.is_contiguous():
            raise EngineError("partials must be contiguous int64 residues")
        polys = part.numel() // ((level + 1) * self.engine.N)
        _lib.check(self.engine._lib.vr_sum_partials(self.engine.handle, part.data_ptr(), polys, level, root))

    def close(self) -> None:
        _lib.check(self.engine._lib.vr_comm_destroy(self.engine.handle))


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) share of n items for ``rank`` of ``world``."""
    if world < 1 or not 0 <= rank < world:
        raise EngineError(f"bad rank {rank} of {world}")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def matmul_nonce_plan(nb: int, n: int, k: int, base: int = 0) -> tuple[list[int], int]:
    """Nonces a single-GPU run assigns: row block b column k -> base + b*n + k; right k -> base + nb*n + k."""
    return [base + b * n + k for b in range(nb)], base + nb * n + k


def encode_operands_sharded(engine: CkksEngine, a_blocks, b, lo: int, hi: int, nonce_base: int = 0):
    """Encrypt only columns k in [lo, hi) of every row block of A and rows k of B.

    a_blocks: list of (m x n) row blocks; b: (n x p).  Returns (lefts, right) holding the local
    ciphertexts with the nonces of an unsharded encode_left/encode_right sequence.
    """
    nb = len(a_blocks)
    a_blocks = [np.atleast_2d(np.asarray(x, dtype=np.float64)) for x in a_blocks]
    b = np.atleast_2d(np.asarray(b, dtype=np.float64))
    m, n = a_blocks[0].shape
    p = b.shape[1]
    lefts = []
    for bi, a in enumerate(a_blocks):
        cts = engine.enc_strided(a, count=hi - lo, nvals=m * p, p=p, sc=1, s1=n, s2=0, offset=lo,
                                 layout=("grid", m, p), nonce0=nonce_base + bi * n + lo)
        lefts.append(ColumnEncodedMatrix(cts, "left", m, hi - lo, p))
    rcts = engine.enc_strided(b, count=hi - lo, nvals=m * p, p=p, sc=p, s1=0, s2=1, offset=lo * p,
                              layout=("grid", m, p), nonce0=nonce_base + nb * n + lo)
    return lefts, ColumnEncodedMatrix(rcts, "right", m, hi - lo, p)


def allreduce_partials(partial: torch.Tensor, group=None) -> torch.Tensor:
    """Sum degree-2 partial residues over ranks (int64, no modular reduction)."""
    import torch.distributed as dist

    if partial.dtype != torch.int64:
        raise EngineError("partials must be int64 residues")
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    return partial


def block_owner(block: int, world: int) -> int:
    """Rank that finishes (relinearises + rescales) row block ``block``: round robin."""
    return block % world


def reduce_partials_to_owners(partial: torch.Tensor, group=None) -> list[int]:
    """Sum each row block's degree-2 partial onto its owner rank only (one reduce per block, int64, no
    modular reduction) and return the blocks this rank owns.  Every rank then relinearises only its
    own blocks instead of all of them: the finishing work is sharded too."""
    import torch.distributed as dist

    if partial.dtype != torch.int64:
        raise EngineError("partials must be int64 residues")
    nb = partial.shape[0]
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return list(range(nb))
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    for b in range(nb):
        owner = block_owner(b, world)
        dst = owner if group is None else dist.get_global_rank(group, owner)
        dist.reduce(partial[b], dst=dst, op=dist.ReduceOp.SUM, group=group)
    return [b for b in range(nb) if block_owner(b, world) == rank]


def matmul_partials(engine: CkksEngine, lefts, right: ColumnEncodedMatrix, out: torch.Tensor | None = None) -> tuple[torch.Tensor, int]:
    """Local degree-2 partial sum [nb][3][l+1][N] (int64 residues) over this rank's k shard (into ``out``
    when given and of the right shape)."""
    nb = len(lefts)
    if nb not in (1, 2, 4):
        raise EngineError("sharded matmul supports 1, 2 or 4 row blocks")
    n = right.n
    for lf in lefts:
        if lf.role != "left" or right.role != "right":
            raise LayoutError("operands must be (left, right) column-encoded shards")
        if lf.n != n or lf.p != right.p or lf.m != right.m:
            raise LayoutError("row blocks must match the right operand's local shard")
    # validated pointer arrays cached on the operands (multicipher._checked_ptrs): a steady-state
    # call does no per-ciphertext Python work (1280 ciphertexts at config 5a)
    infos = [_checked_ptrs(engine, lf) for lf in lefts] + [_checked_ptrs(engine, right)] if n > 0 else []
    lvs = {lv for lv, _ in infos}
    if len(lvs) == 1 and all(p is not None for _, p in infos):
        lv = lvs.pop()
        key = tuple(id(lf) for lf in lefts)
        cat = getattr(right, "_vr_cat", None)
        if cat is None or cat[0] != key:  # the concatenated left table, cached with these row blocks
            cat = (key, _lib.ptr_array([p for _, ps in infos[:-1] for p in ps]), list(lefts))
            object.__setattr__(right, "_vr_cat", cat)
        lptrs = cat[1]
        rptrs = getattr(right, "_vr_ptrs").arr
    else:
        allc = [c for lf in lefts for c in lf.cts] + list(right.cts)
        lv = min(c.level for c in allc) if allc else engine.L
        allc = [engine.adjust(c, lv) for c in allc]
        lptrs = _lib.ptr_array([c.ptr() for c in allc[: nb * n]])
        rptrs = _lib.ptr_array([c.ptr() for c in allc[nb * n:]])
    if lv < 1:
        raise EngineError("multiplicative depth exhausted")
    shape = (nb, 3, lv + 1, engine.N)
    part = out if out is not None and tuple(out.shape) == shape else torch.empty(shape, dtype=torch.int64, device=engine.device)
    if n > 0:
        _lib.check(engine._lib.vr_tensor_sum(engine.handle, lptrs, rptrs, n, nb, lv, _lib.row_ptrs(part, nb)))
    else:
        part.zero_()
    engine._meter.mul_count += nb * n
    engine._meter.add_count += nb * max(n - 1, 0)
    return part, lv


def matmul_finish(engine: CkksEngine, part: torch.Tensor, level: int, m: int, p: int, reduced: bool = False) -> list[Ciphertext]:
    """Summed partials -> mod q (unless already ``reduced``) -> one fused relinearisation + rescale per row block."""
    nb = part.shape[0]
    lib = engine._lib
    if not reduced:
        _lib.check(lib.vr_mod_reduce(engine.handle, part.data_ptr(), nb * 3, level))
    out = torch.empty((nb, 2, level, engine.N), dtype=torch.int64, device=engine.device)
    _lib.check(lib.vr_relin_rescale(engine.handle, _lib.row_ptrs(part, nb),
                                    _lib.row_ptrs(out, nb), nb, level))
    engine._observe(engine.L - level + 1)
    return [Ciphertext.at(out, b, level - 1, engine.scales[level - 1], engine.L - level + 1, ("grid", m, p), engine._id)
            for b in range(nb)]


def matmul_outer_sharded(engine: CkksEngine, lefts, right: ColumnEncodedMatrix, group=None) -> list[Ciphertext]:
    """Distributed matmul_outer: local tensor-sum, one int64 all-reduce, mod q, relin + rescale."""
    part, lv = matmul_partials(engine, lefts, right)
    allreduce_partials(part, group)
    return matmul_finish(engine, part, lv, right.m, right.p)


def matmul_outer_sharded_owned(engine: CkksEngine, lefts, right: ColumnEncodedMatrix, group=None,
                               comm: NativeComm | None = None) -> dict[int, Ciphertext]:
    """Distributed matmul_outer with the finish sharded as well: local tensor-sum, per-block reduce to the
    block's owner, then each rank relinearises + rescales only the blocks it owns ({block: ciphertext};
    empty on ranks that own none).  Residues are identical to matmul_outer_sharded's.  With ``comm`` the
    reduce runs on the library's own NCCL communicator (vr_sum_partials), else on torch.distributed."""
    ring = _partials_buffer(engine, len(lefts), right) if engine.async_drivers else None
    part, lv = matmul_partials(engine, lefts, right, out=ring[0] if ring else None)
    if comm is not None:
        nb = part.shape[0]
        for b in range(nb):
            comm.sum_partials(part[b], lv, root=block_owner(b, comm.world) if comm.world > 1 else -1)
        mine = [b for b in range(nb) if block_owner(b, comm.world) == comm.rank]
        reduced = True
    else:
        mine = reduce_partials_to_owners(part, group)
        # one rank: nothing was summed, the tensor sum's own output is already reduced mod q
        import torch.distributed as dist
        reduced = not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1
    if not mine:
        return {}
    sub = part if len(mine) == part.shape[0] else part[mine].contiguous()
    return dict(zip(mine, _finish_async(engine, sub, lv, right.m, right.p, reduced, ring if sub is part else None)))


def _partials_buffer(engine: CkksEngine, nb: int, right: ColumnEncodedMatrix):
    """Two alternating partial-sum buffers per engine and shape: the tensor sum of product i+1 writes one
    while the side stream still relinearises product i from the other (it first waits for the side
    stream's use of its buffer two products ago).  Fresh allocations per product would be recorded on
    the side stream, and the caching allocator would then fall back to synchronous cudaMalloc calls."""
    lv = min((c.level for c in right.cts), default=engine.L)
    key = ("partials", nb, lv)
    ring = engine._ext_streams.get(key)
    if ring is None:
        ring = engine._ext_streams[key] = {"i": 0, "bufs": [torch.empty((nb, 3, lv + 1, engine.N), dtype=torch.int64,
                                                                        device=engine.device) for _ in range(2)],
                                           "done": [None, None]}
    i = ring["i"]
    ring["i"] = 1 - i
    done = ring["done"][i]
    if done is not None:
        torch.cuda.current_stream(engine.device).wait_event(done)
    return ring["bufs"][i], ring, i


def _finish_async(engine: CkksEngine, part: torch.Tensor, level: int, m: int, p: int, reduced: bool, ring=None) -> list[Ciphertext]:
    """matmul_finish on the engine's side stream: the latency-bound relinearisation of this product
    overlaps the next product's streaming tensor sum (config 5a issues them back to back).  The
    results are pending on the side stream; any read waits for it (Ciphertext._ready)."""
    if not engine.async_drivers:
        return matmul_finish(engine, part, level, m, p, reduced)
    side = engine._side_stream()
    cur = torch.cuda.current_stream(engine.device)
    side.wait_stream(cur)
    with torch.cuda.stream(side):
        outs = matmul_finish(engine, part, level, m, p, reduced)
    if ring is not None:  # the persistent buffer is free again once the side stream passes this point
        _, state, i = ring
        ev = state["done"][i] or torch.cuda.Event()
        ev.record(side)
        state["done"][i] = ev
    else:
        part.record_stream(side)
    for ct in outs:
        ct._pending = side
    return outs


def image_groups(n_images: int, group: int, rank: int, world: int) -> list[tuple[int, int]]:
    """Image index ranges [lo, hi) of the groups of ``group`` images owned by ``rank``."""
    n_groups = (n_images + group - 1) // group
    g_lo, g_hi = shard_range(n_groups, rank, world)
    return [(g * group, min(n_images, (g + 1) * group)) for g in range(g_lo, g_hi)]
