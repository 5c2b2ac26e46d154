"""World-size-2 tests of the multi-GPU host logic on CPU (gloo): k sharding, nonce
plan and the int64 all-reduce of degree-2 partials give residues bit-identical to
the unsharded HE matmul; image-group sharding covers every image exactly once.
The per-rank partials come from the CPU oracle (the checker); the sharding,
nonce plan and reduction are the product's (paper_2512_18646_b200/dist.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_18646_b200.dist import (allreduce_partials, block_owner, image_groups, matmul_nonce_plan,
                                        reduce_partials_to_owners, shard_range)

SLOTS, BITS, DELTA, SEED = 64, (60, 40, 40), 40, 7
NB, M, N_K, P = 2, 4, 6, 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs():
    rng = np.random.default_rng(11)
    a = [rng.uniform(-1, 1, (M, N_K)) for _ in range(NB)]
    b = rng.uniform(-1, 1, (N_K, P))
    return a, b


def _oracle():
    from oracle.engine import OracleEngine

    return OracleEngine(SLOTS, BITS, delta=DELTA, seed=SEED)


def _encrypt(o, a, b, ks):
    """oracle ciphertexts for columns ks with the single-GPU nonce plan"""
    L, R = {}, {}
    for k in ks:
        lnon, rnon = matmul_nonce_plan(NB, N_K, k)
        for bi in range(NB):
            o.nonce = lnon[bi]
            L[(bi, k)] = o.enc(np.repeat(a[bi][:, k], P))
        o.nonce = rnon
        R[k] = o.enc(np.tile(b[k, :], M))
    return L, R


def _partial(o, L, R, ks):
    q = np.array(o.q[: o.L + 1], dtype=object)
    out = np.zeros((NB, 3, o.L + 1, o.N), dtype=object)
    for bi in range(NB):
        for k in ks:
            d3 = o.c.tensor(L[(bi, k)].data, R[k].data).astype(object)
            out[bi] = (out[bi] + d3) % q[None, :, None]
    return out.astype(np.int64)


def _finish(o, summed):
    q = np.array(o.q[: o.L + 1], dtype=np.uint64)
    res = []
    for bi in range(NB):
        d3 = (summed[bi].astype(np.uint64) % q[None, :, None]).astype(np.uint64)
        res.append(o.c.relin_rescale(np.ascontiguousarray(d3)))
    return res


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = _inputs()
        o = _oracle()
        lo, hi = shard_range(N_K, rank, world)
        L, R = _encrypt(o, a, b, range(lo, hi))
        part = torch.from_numpy(_partial(o, L, R, range(lo, hi)))
        allreduce_partials(part)
        res = _finish(o, part.numpy())
        q.put((rank, [r.copy() for r in res]))
    finally:
        dist.destroy_process_group()


def test_shard_range_partition():
    for n in (1, 7, 256):
        for world in (1, 2, 3, 4, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [h - l for l, h in parts]
            assert max(sizes) - min(sizes) <= 1


def test_image_groups_cover_once():
    for world in (1, 2, 4, 8):
        seen = []
        for r in range(world):
            for lo, hi in image_groups(512, 16, r, world):
                seen.extend(range(lo, hi))
        assert sorted(seen) == list(range(512))


def test_sharded_matmul_bit_exact_world2():
    a, b = _inputs()
    o = _oracle()
    L, R = _encrypt(o, a, b, range(N_K))
    want = _finish(o, _partial(o, L, R, range(N_K)))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in (0, 1):
        for bi in range(NB):
            np.testing.assert_array_equal(got[rank][bi], want[bi])
    dec = o.dec(type("C", (), {"data": want[0], "scale": o.scales[o.L - 1]})())
    np.testing.assert_allclose(dec[: M * P].reshape(M, P), a[0] @ b, atol=1e-3)


def _worker_owned(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = _inputs()
        o = _oracle()
        lo, hi = shard_range(N_K, rank, world)
        L, R = _encrypt(o, a, b, range(lo, hi))
        part = torch.from_numpy(_partial(o, L, R, range(lo, hi)))
        mine = reduce_partials_to_owners(part)
        res = _finish(o, part.numpy())  # only the owned blocks hold the full sum
        q.put((rank, mine, {bi: res[bi].copy() for bi in mine}))
    finally:
        dist.destroy_process_group()


def test_owner_reduce_bit_exact_world2():
    """Per-block reduce to the owner rank (the finish sharded over ranks): every block is owned by
    exactly one rank and its finished residues equal the unsharded result."""
    a, b = _inputs()
    o = _oracle()
    L, R = _encrypt(o, a, b, range(N_K))
    want = _finish(o, _partial(o, L, R, range(N_K)))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_owned, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    owned = sorted(bi for _, mine, _ in got for bi in mine)
    assert owned == list(range(NB))
    for rank, mine, res in got:
        assert mine == [bi for bi in range(NB) if block_owner(bi, 2) == rank]
        for bi in mine:
            np.testing.assert_array_equal(res[bi], want[bi])
