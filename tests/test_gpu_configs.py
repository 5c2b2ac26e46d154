"""BASELINE configs on the GPU: bit-exact residues against the CPU oracle where
the oracle finishes in seconds (configs 1, 2 and reduced-size config 4 with the
config-4 parameters), and decoded values within 1e-3 of the plaintext result at
full size (size-independent check)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.engine import OracleEngine  # noqa: E402
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer  # noqa: E402
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
