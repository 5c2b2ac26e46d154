"""BASELINE configs on the GPU: bit-exact residues against the CPU oracle where
the oracle finishes in seconds (configs 1, 2 and reduced-size config 4 with the
config-4 parameters), and decoded values within 1e-3 of the plaintext result at
full size (size-independent check)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.engine import OracleEngine  # noqa: E402
from paper_2512_18646_b200 import (CkksEngine, LayoutError, config_params, encode_left, encode_right, matmul_outer,  # noqa: E402
                                   matmul_outer_many)
from paper_2512_18646_b200.cnn import conv_layer, decode_layer, encode_images  # noqa: E402
from tools.workloads import ACT4, cfg4, cfg_matmul, conv_plain, poly_plain  # noqa: E402

TOL = 1e-3


@pytest.mark.parametrize("cfg", [1, 2])
def test_matmul_configs_bit_exact(cfg):
    p = config_params(cfg)
    g, o = CkksEngine(p), OracleEngine.from_params(p)
    a, b = cfg_matmul(cfg)
    dim = a.shape[0]
    out = matmul_outer(g, encode_left(g, a, dim), encode_right(g, b, dim))
    oL = [o.enc(np.repeat(a[:, k], dim)) for k in range(dim)]
    oR = [o.enc(np.tile(b[k, :], dim)) for k in range(dim)]
    want = o.matmul_outer_blocks([oL], oR)[0]
    np.testing.assert_array_equal(out.ct.residues(), want.data)
    np.testing.assert_allclose(out.decode(g), a @ b, atol=TOL)
    assert out.ct.depth == 1


@pytest.mark.parametrize("cfg,dim,count", [(1, 8, 8), (1, 8, 3), (2, 64, 2), (1, 5, 4)])
def test_matmul_outer_many_equals_separate_products(cfg, dim, count):
    """vr_matmul_outer_many: `count` independent products in one launch sequence -- residues equal the
    separate matmul_outer calls and the CPU oracle (multicipher.py:88-103 once per pair); meter and
    depth as for separate calls."""
    p = config_params(cfg)
    g, o = CkksEngine(p), OracleEngine.from_params(p)
    rng = np.random.default_rng(100 + cfg)
    mats = [rng.uniform(-1, 1, (2, dim, dim)) for _ in range(count)]
    pairs = [(encode_left(g, a, dim), encode_right(g, b, dim)) for a, b in mats]
    before = g.meter_snapshot()
    outs = matmul_outer_many(g, pairs)
    d = g.meter_snapshot().delta_since(before)
    assert (d.mul_count, d.add_count) == (count * dim, count * (dim - 1))
    assert len(outs) == count
    for i, ((a, b), out) in enumerate(zip(mats, outs)):
        single = matmul_outer(g, *pairs[i])
        np.testing.assert_array_equal(out.ct.residues(), single.ct.residues())
        np.testing.assert_allclose(out.decode(g), a @ b, atol=TOL)
        assert out.ct.depth == 1 and out.ct.level == single.ct.level
    # oracle: the encryptions consumed nonces pair by pair (left then right), as on the GPU
    for i, (a, b) in enumerate(mats[:2]):
        oL = [o.enc(np.repeat(a[:, k], dim)) for k in range(dim)]
        oR = [o.enc(np.tile(b[k, :], dim)) for k in range(dim)]
        want = o.matmul_outer_blocks([oL], oR)[0]
        np.testing.assert_array_equal(outs[i].ct.residues(), want.data)
    # twice with the same operands (the replayed graph) gives the same residues
    again = matmul_outer_many(g, pairs)
    for x, y in zip(outs, again):
        np.testing.assert_array_equal(x.ct.residues(), y.ct.residues())


def test_matmul_outer_many_validation():
    g = CkksEngine(config_params(1))
    a = np.random.default_rng(5).uniform(-1, 1, (8, 8))
    l8, r8 = encode_left(g, a, 8), encode_right(g, a, 8)
    l4, r4 = encode_left(g, a[:4, :4], 4), encode_right(g, a[:4, :4], 4)
    assert matmul_outer_many(g, []) == []
    with pytest.raises(LayoutError):
        matmul_outer_many(g, [(r8, l8)])
    with pytest.raises(LayoutError):
        matmul_outer_many(g, [(l8, r8), (l4, r4)])
    with pytest.raises(LayoutError):
        matmul_outer_many(g, [(l8, r4)])


def test_cfg4_reduced_bit_exact():
    """config-4 parameters (N=2^15, 8 primes, scale 2^45) on 2 small padded images, 2 filters."""
    p = config_params(4)
    g, o = CkksEngine(p), OracleEngine.from_params(p)
    rng = np.random.default_rng(3)
    imgs = rng.uniform(0, 1, (2, 3, 10, 10))
    w = rng.normal(0, 0.05, (2, 3, 3, 3))
    bias = np.array([0.0, 0.1])
    chans = encode_images(g, imgs, padding=1)
    ys = conv_layer(g, chans, w, bias, activation=ACT4)
    padded = np.pad(imgs, ((0, 0), (0, 0), (1, 1), (1, 1)))
    X = [o.enc(padded[:, c, :, j].reshape(-1)) for c in range(3) for j in range(12)]
    oy = o.conv_columns_multi(X, 3, 12, w, bias, range(10), 2, 12, 10)
    for f in range(2):
        for j in range(10):
            ref = o.poly_activation(oy[f * 10 + j], ACT4)
            np.testing.assert_array_equal(ys[f].cts[j].residues(), ref.data)
    got = decode_layer(g, ys)
    np.testing.assert_allclose(got, poly_plain(conv_plain(imgs, w, bias, padding=1), ACT4), atol=TOL)


def test_cfg4_full_size_decoded():
    """the full config-4 layer (16 images, 16 filters, 3x224x224, padding 1) vs the plaintext CNN."""
    imgs, w, b = cfg4(16)
    g = CkksEngine(config_params(4))
    chans = encode_images(g, imgs, padding=1)
    ys = conv_layer(g, chans, w, b, activation=ACT4)
    got = decode_layer(g, ys)
    want = poly_plain(conv_plain(imgs, w, b, padding=1), ACT4)
    assert got.shape == (16, 16, 224, 224)
    assert float(np.max(np.abs(got - want))) < TOL
    assert all(ct.depth == 3 for y in ys for ct in y.cts)


def _oracle_cfg3(o, imgs, w, w1, w2):
    """Oracle restatement of paper_2512_18646_b200.cnn.cnn_cfg3 (same ciphertexts, same op order)."""
    m, h, wd = imgs.shape
    F, _, k, _ = w.shape
    cols = list(range(0, wd - k + 1, 2))
    rows = list(range(0, h - k + 1, 2))
    X = [o.enc(imgs[:, :, j].reshape(-1)) for j in range(wd)]
    conv = o.conv_columns_multi(X, 1, wd, w, np.zeros(F), cols, m, h, h - k + 1)
    feats = [o.mul(c, c) for c in conv]
    lv = feats[0].level
    S, nr, no, ny = o.slots, len(rows), len(cols), w1.shape[0]
    slot_idx = (np.arange(m)[:, None] * h + np.asarray(rows)[None, :]).reshape(-1)

    def dense(xs, mask_rows, ny_):
        lvx = xs[0].level
        outs = []
        for u in range(ny_):
            acc = None
            for j, x in enumerate(xs):
                term = o.c.mul_plain(x.data, o.c.encode(mask_rows[u * len(xs) + j], lvx, o.scales[lvx]))
                acc = term if acc is None else o.c.add(acc, term)
            outs.append(type(xs[0])(o.c.rescale(acc), lvx - 1, o.scales[lvx - 1]))
        return outs

    masks = np.zeros((ny, F * no, S))
    for f in range(F):
        for oc in range(no):
            masks[:, f * no + oc, slot_idx] = np.tile(w1[:, f * nr * no + np.arange(nr) * no + oc], (1, m))
    hid = dense(feats, masks.reshape(-1, S), ny)
    T1 = hid
    T2 = [o.add(t, o.rot(t, 2)) for t in T1]
    T4 = [o.add(t, o.rot(t, 4)) for t in T2]
    T8 = [o.add(t, o.rot(t, 8)) for t in T4]
    tot = [o.add(o.add(a, o.rot(t1, 24)), o.rot(t4, 16)) for a, t1, t4 in zip(T8, T1, T4)]
    sq = [o.mul(t, t) for t in tot]
    return dense(sq, np.repeat(w2.reshape(-1, 1), S, axis=1), w2.shape[0])


def test_cfg3_reduced_bit_exact():
    from paper_2512_18646_b200.cnn import cnn_cfg3
    from tools.workloads import cfg3

    imgs, w, w1, w2 = cfg3()
    imgs, w1, w2 = imgs[:3], w1[:4], w2[:, :4]
    p = config_params(3)
    g, o = CkksEngine(p), OracleEngine.from_params(p)
    logits = cnn_cfg3(g, imgs, w, w1, w2)
    want = _oracle_cfg3(o, imgs, w, w1, w2)
    for gl, ol in zip(logits, want):
        assert gl.level == 0
        np.testing.assert_array_equal(gl.residues(), ol.data)


def test_cfg3_full_size_decoded():
    from paper_2512_18646_b200.cnn import cnn_cfg3, decode_logits
    from tools.workloads import cfg3, cfg3_plain

    imgs, w, w1, w2 = cfg3()
    g = CkksEngine(config_params(3))
    logits = cnn_cfg3(g, imgs, w, w1, w2)
    got = decode_logits(g, logits, 64, 28)
    want = cfg3_plain(imgs, w, w1, w2)
    assert got.shape == (64, 10)
    assert float(np.max(np.abs(got - want))) < TOL
    assert all(c.level == 0 and c.depth == 5 for c in logits)


@pytest.mark.parametrize("slots,nx,ny", [(1024, 131, 3), (4, 5, 3)])
def test_dense_columns_bit_exact(slots, nx, ny):
    """k_pt_matvec: more inputs than one shared-memory pointer chunk (128), an odd output count,
    and a ring smaller than one CTA's coefficient tile; residues vs the oracle's cmul/add/rescale."""
    from paper_2512_18646_b200 import EngineParams
    from paper_2512_18646_b200.cnn import dense_columns, encode_plain_batch

    p = EngineParams(slots=slots, prime_bits=(60, 40, 40), delta=40, seed=5)
    g, o = CkksEngine(p), OracleEngine.from_params(p)
    rng = np.random.default_rng(11)
    xs = rng.uniform(-1, 1, (nx, slots))
    ws = rng.uniform(-1, 1, (ny * nx, slots))
    gx, ox = [g.enc(v) for v in xs], [o.enc(v) for v in xs]
    lv = gx[0].level
    ys = dense_columns(g, gx, encode_plain_batch(g, ws, lv, g.scales[lv]), ny)
    for u in range(ny):
        acc = None
        for j in range(nx):
            term = o.c.mul_plain(ox[j].data, o.c.encode(ws[u * nx + j], lv, o.scales[lv]))
            acc = term if acc is None else o.c.add(acc, term)
        np.testing.assert_array_equal(ys[u].residues(), o.c.rescale(acc))
        np.testing.assert_allclose(g.dec(ys[u]), (xs * ws[u * nx:(u + 1) * nx]).sum(axis=0), atol=TOL)
