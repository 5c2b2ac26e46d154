"""Self-consistency of the CPU RNS-CKKS residue oracle and its decoded-value
agreement with the reference algorithm (oracle/sim.py, itself pinned to the
reference's outputs).  CPU only."""

import numpy as np
import pytest

from oracle import ckks as O
from oracle import sim
from oracle.engine import OracleEngine
from paper_2512_18646_b200.params import gen_primes as product_gen_primes


def negacyclic(a, b, q):
    n = len(a)
    out = [0] * n
    for i in range(n):
        ai = int(a[i])
        for j in range(n):
            v = ai * int(b[j])
            k = i + j
            if k >= n:
                out[k - n] = (out[k - n] - v) % q
            else:
                out[k] = (out[k] + v) % q
    return np.array(out, dtype=np.uint64)


@pytest.mark.parametrize("log_n", [2, 3, 5, 7])
def test_ntt_is_negacyclic_convolution(log_n):
    primes = O.gen_primes(log_n, [60, 40, 45, 60])
    c = O.OracleCkks(log_n, primes, seed=1)
    rng = np.random.default_rng(log_n)
    for pidx in range(len(primes)):
        q = int(primes[pidx])
        a = rng.integers(0, q, 1 << log_n, dtype=np.uint64)
        b = rng.integers(0, q, 1 << log_n, dtype=np.uint64)
        A, B = c.ntt(a, pidx), c.ntt(b, pidx)
        np.testing.assert_array_equal(c.intt(A, pidx), a)
        prod = np.array([(int(x) * int(y)) % q for x, y in zip(A, B)], dtype=np.uint64)
        np.testing.assert_array_equal(c.intt(prod, pidx), negacyclic(a, b, q))


@pytest.mark.parametrize("log_n", [3, 6, 13, 14, 15])
def test_prime_generation_matches_product(log_n):
    bits = [60, 40, 40, 45, 45, 60]
    assert [int(x) for x in O.gen_primes(log_n, bits)] == product_gen_primes(log_n, bits)


def test_encode_is_canonical_embedding():
    log_n = 6
    n = 1 << log_n
    c = O.OracleCkks(log_n, O.gen_primes(log_n, [60, 40, 60]), seed=3)
    z = np.random.default_rng(1).uniform(-1, 1, n // 2)
    m = c.encode_coeffs(z, 2.0 ** 40)
    zeta = np.exp(1j * np.pi / n)
    ev = np.array([sum(int(m[k]) * zeta ** (pow(5, j, 2 * n) * k) for k in range(n)) for j in range(n // 2)]) / 2.0 ** 40
    np.testing.assert_allclose(ev.real, z, atol=1e-9)
    np.testing.assert_allclose(ev.imag, 0, atol=1e-9)
    np.testing.assert_allclose(c.decode_coeffs(m, 2.0 ** 40).real, z, atol=1e-9)


def test_automorphism_perm_matches_coefficient_map():
    log_n = 5
    n = 1 << log_n
    primes = O.gen_primes(log_n, [60, 40, 60])
    c = O.OracleCkks(log_n, primes, seed=3)
    q = int(primes[1])
    a = np.random.default_rng(2).integers(0, q, n, dtype=np.uint64)
    for g in (5, 25, 2 * n - 1):
        sig = np.zeros(n, dtype=np.uint64)
        for k in range(n):
            e = (k * g) % (2 * n)
            if e < n:
                sig[e] = a[k]
            else:
                sig[e - n] = (q - int(a[k])) % q
        perm = c.galois_perm(g)
        A = c.ntt(a, 1)
        np.testing.assert_array_equal(A[perm], c.ntt(sig, 1))


@pytest.mark.parametrize("enc", ["public", "secret"])
def test_primitives_decode(enc):
    e = OracleEngine(16, (60, 40, 40, 40), delta=40, seed=9, encryption=enc)
    rng = np.random.default_rng(5)
    x, y = rng.uniform(-1, 1, 16), rng.uniform(-1, 1, 16)
    a, b = e.enc(x), e.enc(y)
    np.testing.assert_allclose(e.dec(a), x, atol=1e-6)
    np.testing.assert_allclose(e.dec(e.add(a, b)), x + y, atol=1e-6)
    ab = e.mul(a, b)
    assert ab.level == 2 and ab.depth == 1
    np.testing.assert_allclose(e.dec(ab), x * y, atol=1e-6)
    np.testing.assert_allclose(e.dec(e.add(ab, a)), x * y + x, atol=1e-6)  # cross-level add
    for s in (1, -1, 5, 16, -17):
        np.testing.assert_allclose(e.dec(e.rot(a, s)), np.roll(x, -s), atol=1e-6)
    np.testing.assert_allclose(e.dec(e.cmul(np.full(16, 0.5), a)), 0.5 * x, atol=1e-6)
    mask = (np.arange(16) % 3 == 0).astype(float)
    np.testing.assert_allclose(e.dec(e.cmul(mask, a)), mask * x, atol=1e-6)


def test_rescale_rounds():
    e = OracleEngine(8, (60, 40), delta=40, seed=1)
    ct = e.enc(np.full(8, 0.75))
    out = e.c.rescale(e.c.mul_scalar(ct.data, 2 ** 20))
    np.testing.assert_allclose(e.c.decrypt_decode(out, 2.0 ** 60 / e.q[1]), 0.75, atol=1e-5)


def test_matmul_outer_fused_matches_reference_algorithm(golden):
    for idx in (2, 3, 5, 6):
        a, b = golden[f"mm{idx}_a"], golden[f"mm{idx}_b"]
        m, n = a.shape
        p = b.shape[1]
        slots = max(2, 1 << (m * p - 1).bit_length())
        e = OracleEngine(slots, (60, 40, 40), delta=40, seed=idx)
        L = [e.enc(np.repeat(a[:, k], p)) for k in range(n)]
        R = [e.enc(np.tile(b[k, :], m)) for k in range(n)]
        out = e.matmul_outer_blocks([L], R)[0]
        got = e.dec(out)[: m * p].reshape(m, p)
        np.testing.assert_allclose(got, golden[f"mm{idx}_c"], atol=1e-3)


def test_conv_fused_matches_reference_algorithm(golden):
    for idx in range(5):
        imgs, w, bias = golden[f"cv{idx}_img"], golden[f"cv{idx}_w"], float(golden[f"cv{idx}_bias"][0])
        m, h, wd = imgs.shape
        k = w.shape[0]
        slots = max(2, 1 << (m * h - 1).bit_length())
        e = OracleEngine(slots, (60, 40, 40), delta=40, seed=idx)
        X = [e.enc(imgs[:, :, j].reshape(-1)) for j in range(wd)]
        out_h = h - k + 1
        Y = e.conv_columns_multi(X, 1, wd, w[None, None], [bias], range(wd - k + 1), m, h, out_h)
        got = np.stack([e.dec(y) for y in Y], axis=-1)  # [slots][out_w]
        for b in range(m):
            np.testing.assert_allclose(got[b * h: b * h + out_h], golden[f"cv{idx}_out"][b], atol=1e-3)
            # masked (invalid) rows are zero like the reference's
            np.testing.assert_allclose(got[b * h + out_h: (b + 1) * h], 0.0, atol=1e-3)


def test_poly_fused_matches_reference_algorithm(golden):
    for idx in range(4):
        x, coeffs = golden[f"pa{idx}_x"], golden[f"pa{idx}_coeffs"]
        e = OracleEngine(16, (60, 40, 40, 40), delta=40, seed=idx)
        out = e.poly_activation(e.enc(x), coeffs)
        assert out.depth == 2 and out.level == 1
        np.testing.assert_allclose(e.dec(out), golden[f"pa{idx}_out"], atol=1e-3)


def test_keyswitch_identity():
    """ks(c) with the relin key decrypts to c * s^2 (checked through relinearisation)."""
    e = OracleEngine(16, (60, 40, 40), delta=40, seed=4)
    x = np.random.default_rng(3).uniform(-1, 1, 16)
    a = e.enc(x)
    d3 = e.c.tensor(a.data, a.data)
    relin = e.c.relin(d3)
    m3 = e.c.decrypt_coeffs(d3)
    m2 = e.c.decrypt_coeffs(relin)
    assert np.max(np.abs(m3 - m2)) < 2 ** 20  # key-switch noise only
