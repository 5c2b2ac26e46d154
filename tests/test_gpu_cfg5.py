"""Config 5 against the CPU residue oracle at the BASELINE shapes.

* 5a (multicipher.py:88-103): the full 256x256 HE matmul -- 4 row
  blocks x 256 column ciphertexts, N = 2^15, l = 8 -- through matmul_outer_blocks,
  through the k-sharded path with virtual ranks (int64 partial sums, like the NCCL
  reduce) and through the owner-reduce variant: every result bit-identical to the
  C oracle's fused matmul_outer on the same input residues; a sample of the input
  encryptions bit-identical to the oracle's own encryptions with the same nonces.
* 5b (multicipher.py:106-162 + pipeline.py:180-197): the 64-images-per-ciphertext
  geometry (stride 226 = 224 rows + padding, 14,464 of 16,384 slots) with the
  config-4 layer (3 channels, 3x3 taps, padding 1, activation 0.125x^2+0.5x+0.25),
  columns reduced to 6: residues bit-identical to the oracle's conv_columns_multi +
  poly_activation, decoded within 1e-3 of the plaintext CNN.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.engine import OCt, OracleEngine  # noqa: E402
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer_blocks  # noqa: E402
from paper_2512_18646_b200.cnn import conv_layer, decode_layer, encode_images  # noqa: E402
from paper_2512_18646_b200.dist import (encode_operands_sharded, matmul_finish, matmul_outer_sharded_owned,  # noqa: E402
                                        matmul_partials, shard_range)
from tools.workloads import ACT4, cfg_matmul, conv_plain, poly_plain  # noqa: E402

TOL = 1e-3


def _oct(ct):
    return OCt(ct.residues(), ct.level, ct.scale, ct.depth)


def test_cfg5a_full_size_bit_exact_vs_oracle():
    p = config_params(5)
    g, o = CkksEngine(p), OracleEngine.from_params(p)
    a, b = cfg_matmul(5)
    blocks = [a[64 * i: 64 * (i + 1)] for i in range(4)]
    lefts = [encode_left(g, blk, 256) for blk in blocks]  # nonces b*256 + k
    right = encode_right(g, b, 64)  # nonces 1024 + k
    # input encryptions: the oracle's own, same nonces (first/last column of a block, the right operand)
    for cts, k, vals, nonce in [(lefts[0].cts, 0, np.repeat(blocks[0][:, 0], 256), 0),
                                (lefts[3].cts, 255, np.repeat(blocks[3][:, 255], 256), 3 * 256 + 255),
                                (right.cts, 17, np.tile(b[17, :], 64), 1024 + 17)]:
        o.nonce = nonce
        np.testing.assert_array_equal(cts[k].residues(), o.enc(vals).data)
    # the oracle's fused matmul_outer on the GPU's input residues
    want = o.matmul_outer_blocks([[_oct(c) for c in lf.cts] for lf in lefts], [_oct(c) for c in right.cts])
    want = [w.data for w in want]
    got = matmul_outer_blocks(g, lefts, right)
    for gb, wb in zip(got, want):
        np.testing.assert_array_equal(gb.residues(), wb)
    dec = np.concatenate([g.dec(c)[: 64 * 256].reshape(64, 256) for c in got])
    assert float(np.max(np.abs(dec - a @ b))) < TOL
    del lefts, right, got
    # k-sharded over 4 virtual ranks: partial sums added like the NCCL int64 reduce
    total, lv = None, None
    for rank in range(4):
        lo, hi = shard_range(256, rank, 4)
        ls, rs = encode_operands_sharded(g, blocks, b, lo, hi)
        part, lv = matmul_partials(g, ls, rs)
        total = part if total is None else total + part
        del ls, rs
    for ob, wb in zip(matmul_finish(g, total, lv, 64, 256), want):
        np.testing.assert_array_equal(ob.residues(), wb)
    del total
    # owner-reduce variant, one rank owning all four blocks
    ls, rs = encode_operands_sharded(g, blocks, b, 0, 256)
    owned = matmul_outer_sharded_owned(g, ls, rs)
    assert sorted(owned) == [0, 1, 2, 3]
    for bi, wb in enumerate(want):
        np.testing.assert_array_equal(owned[bi].residues(), wb)


def test_cfg5b_geometry_bit_exact_vs_oracle():
    """64 images per column ciphertext at the config-5b stride (226 padded rows); 6 columns, 4 filters."""
    p = config_params(5)
    g, o = CkksEngine(p), OracleEngine.from_params(p)
    rng = np.random.default_rng(4)
    m, h, w_cols, F = 64, 224, 6, 4
    imgs = rng.uniform(0, 1, (m, 3, h, w_cols))
    w = rng.normal(0, 0.05, (F, 3, 3, 3))
    bias = np.zeros(F)
    chans = encode_images(g, imgs, padding=1)
    assert chans[0].stride == 226 and m * chans[0].stride == 14464
    ys = conv_layer(g, chans, w, bias, activation=ACT4)
    padded = np.pad(imgs, ((0, 0), (0, 0), (1, 1), (1, 1)))
    W = w_cols + 2
    X = [o.enc(padded[:, c, :, j].reshape(-1)) for c in range(3) for j in range(W)]  # same nonce order
    oy = o.conv_columns_multi(X, 3, W, w, bias, range(w_cols), m, 226, h)
    for f in range(F):
        for j in range(w_cols):
            ref = o.poly_activation(oy[f * w_cols + j], ACT4)
            np.testing.assert_array_equal(ys[f].cts[j].residues(), ref.data)
    got = decode_layer(g, ys)
    want = poly_plain(conv_plain(imgs, w, bias, padding=1), ACT4)
    assert got.shape == want.shape == (m, F, h, w_cols)
    assert float(np.max(np.abs(got - want))) < TOL
