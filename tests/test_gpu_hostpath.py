"""The host side of a product (round 2): deferred, host-staged operand encryption
(``vr_encrypt_strided*_host``), lazily materialised ciphertext batches (``CtBatch``), decode tickets
(``vr_decode_submit`` / ``vr_decode_wait``) and pipelined encrypt -> product -> decode loops.  Every
path must give exactly the residues of the plain per-call path (engine.py:193-206,
multicipher.py:62-103 of the reference define the values)."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2512_18646_b200 import (CkksEngine, EngineParams, _lib, encode_image_columns, encode_left,  # noqa: E402
                                   encode_right, matmul_outer)
from paper_2512_18646_b200.engine import CtBatch  # noqa: E402

TOL = 1e-3
PARAMS = EngineParams(slots=1024, prime_bits=(60, 40, 40), delta=40, seed=11)


def _operands(rng, n=8):
    return rng.uniform(-1, 1, (n, n)), rng.uniform(-1, 1, (n, n))


def test_deferred_encryption_matches_the_eager_one():
    """encode_left / encode_right are deferred and launched as ONE host-staged encryption; the
    ciphertexts are bit-identical to eager per-row encryptions with the same nonces."""
    a, b = _operands(np.random.default_rng(0))
    eng = CkksEngine(PARAMS)
    left, right = encode_left(eng, a, 8), encode_right(eng, b, 8)
    assert isinstance(left.cts, CtBatch) and left.cts._items is None  # nothing materialised, nothing launched
    assert len(eng._enc_queue) == 2 or not eng._defer_enc
    got_l = [ct.residues() for ct in left.cts]  # first access launches both operands
    got_r = [ct.residues() for ct in right.cts]
    assert not eng._enc_queue
    ref = CkksEngine(PARAMS)
    want_l = ref.enc_batch([np.repeat(a[:, k], 8) for k in range(8)], nonce0=0)
    want_r = ref.enc_batch([np.tile(b[k, :], 8) for k in range(8)], nonce0=8)
    for g, w in zip(got_l + got_r, want_l + want_r):
        np.testing.assert_array_equal(g, w.residues())


def test_host_array_is_snapshotted():
    """The caller may overwrite its array between encode_* and the deferred launch."""
    a, b = _operands(np.random.default_rng(1))
    eng = CkksEngine(PARAMS)
    a_work, b_work = a.copy(), b.copy()
    left, right = encode_left(eng, a_work, 8), encode_right(eng, b_work, 8)
    a_work[:] = 7.0
    b_work[:] = -3.0
    got = matmul_outer(eng, left, right).decode(eng)
    np.testing.assert_allclose(got, a @ b, atol=TOL)


def test_ct_batch_is_list_like():
    a, _ = _operands(np.random.default_rng(2))
    eng = CkksEngine(PARAMS)
    cts = encode_left(eng, a, 8).cts
    assert len(cts) == 8
    assert [c._idx for c in cts] == list(range(8))
    assert cts[3] is cts[3] and cts[-1]._idx == 7
    assert [c._idx for c in cts[2:4]] == [2, 3]
    assert len(cts + [1]) == 9 and len([0] + cts) == 9
    assert list(cts.pointers()) == [c._ptr for c in cts]
    np.testing.assert_allclose(eng.dec(cts[5])[:64].reshape(8, 8), np.repeat(a[:, 5], 8).reshape(8, 8), atol=TOL)


def test_strided_host_entry_points_match_the_device_form():
    """vr_encrypt_strided_host (C-ABI) == vr_encrypt_strided on a device copy of the same array."""
    eng = CkksEngine(PARAMS)
    lib, h = eng._lib, eng.handle
    rng = np.random.default_rng(3)
    src = np.ascontiguousarray(rng.uniform(-1, 1, 200))
    count, nvals, p = 4, 48, 6
    out_h = torch.empty((count, 2, eng.L + 1, eng.N), dtype=torch.int64, device="cuda")
    out_d = torch.empty_like(out_h)
    _lib.check(lib.vr_encrypt_strided_host(h, src.ctypes.data, src.size, 5, 7, 6, 1, p, nvals, count, eng.L,
                                           eng.scales[eng.L], 100, out_h.data_ptr()))
    d_src = torch.from_numpy(src).cuda()
    _lib.check(lib.vr_encrypt_strided(h, d_src.data_ptr() + 8 * 5, 7, 6, 1, p, nvals, count, eng.L, eng.scales[eng.L], 100,
                                      out_d.data_ptr()))
    assert torch.equal(out_h, out_d)
    # bad arguments are reported, not dereferenced
    assert lib.vr_encrypt_strided_host(h, src.ctypes.data, 0, 0, 7, 6, 1, p, nvals, count, eng.L, eng.scales[eng.L], 0,
                                       out_h.data_ptr()) != 0
    assert lib.vr_encrypt_strided_host(h, src.ctypes.data, src.size, 0, 7, 6, 1, p, eng.slots + 1, count, eng.L,
                                       eng.scales[eng.L], 0, out_h.data_ptr()) == 1  # CapacityError


def test_decode_tickets_match_blocking_decode():
    """dec_batch_async (library tickets) == dec_batch, for several futures in flight, resolved out of
    order, dropped unresolved, and for results of asynchronous products."""
    rng = np.random.default_rng(4)
    eng = CkksEngine(PARAMS)
    vals = [rng.uniform(-1, 1, 1024) for _ in range(6)]
    cts = [eng.enc(v) for v in vals]
    futs = [eng.dec_batch_async([ct]) for ct in cts]
    for i in (3, 0, 5, 1):
        got = futs[i].result()
        assert got.shape == (1, 1024)
        np.testing.assert_array_equal(got, eng.dec_batch([cts[i]]))
        np.testing.assert_array_equal(futs[i].result(), got)  # a future can be read again
    del futs  # two tickets never waited for: released by the finaliser
    many = eng.dec_batch_async(cts).result()
    np.testing.assert_array_equal(many, eng.dec_batch(cts))
    # selections keep the torch path
    sel = eng.dec_batch_async(cts[:2], select=[0, 5, 9]).result()
    np.testing.assert_array_equal(sel, eng.dec_batch(cts[:2], select=[0, 5, 9]))
    # unknown ticket
    assert eng._lib.vr_decode_wait(eng.handle, 999, None) != 0


def test_pipelined_products_equal_sequential_ones():
    """Several encrypt -> matmul_outer -> decode_async steps in flight: values equal A @ B and the
    residues equal the one-at-a-time run of a second engine with the same seed."""
    rng = np.random.default_rng(5)
    pairs = [_operands(rng) for _ in range(6)]
    eng, ref = CkksEngine(PARAMS), CkksEngine(PARAMS)
    futs, prods = [], []
    for a, b in pairs:
        prod = matmul_outer(eng, encode_left(eng, a, 8), encode_right(eng, b, 8))
        prods.append(prod)
        futs.append(prod.decode_async(eng))
    for (a, b), f, prod in zip(pairs, futs, prods):
        np.testing.assert_allclose(f.result(), a @ b, atol=TOL)
        want = matmul_outer(ref, encode_left(ref, a, 8), encode_right(ref, b, 8))
        ref.join()
        np.testing.assert_array_equal(prod.ct.residues(), want.ct.residues())


def test_operand_reused_on_other_slots():
    """One encrypted operand pair consumed by consecutive products (different slot streams)."""
    a, b = _operands(np.random.default_rng(6))
    eng = CkksEngine(PARAMS)
    left, right = encode_left(eng, a, 8), encode_right(eng, b, 8)
    outs = [matmul_outer(eng, left, right) for _ in range(10)]
    first = outs[0].ct.residues()
    for o in outs[1:]:
        np.testing.assert_array_equal(o.ct.residues(), first)
    np.testing.assert_allclose(outs[-1].decode(eng), a @ b, atol=TOL)


def test_large_sources_keep_the_device_path():
    """Raw arrays above the host-staging limit (images) are uploaded through the pinned torch ring."""
    eng = CkksEngine(EngineParams(slots=4096, prime_bits=(60, 40, 40), delta=40, seed=2))
    imgs = np.random.default_rng(7).uniform(0, 1, (8, 512, 40))  # 1.3 MB > 1 MB
    cei = encode_image_columns(eng, imgs)
    got = eng.dec(cei.cts[3])[: 8 * 512].reshape(8, 512)
    np.testing.assert_allclose(got, imgs[:, :, 3], atol=TOL)
