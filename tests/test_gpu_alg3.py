"""Algorithm 3 (revolver matmul) on the GPU engine: the reference's test_matmul.py cases
(exact equality -> <= 1e-3 decoded error; meter counts and depths exact, pinned by the
reference's own fixtures), and bit-exact residues of the batched GPU path against the
per-iteration loop run on the C residue oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.engine import OracleEngine  # noqa: E402
from paper_2512_18646_b200 import (  # noqa: E402
    EngineError, EngineParams, LayoutError, MatmulPlan, SlotEngine, build_result_filter, encode_revolver,
    encode_row_major, matmul, matmul_tiled, row_shifter)

from conftest import rand_int_matrix  # noqa: E402

TOL = 1e-3
CHAIN = (60, 45, 45, 45, 45)


def make_engine(slots: int) -> SlotEngine:
    return SlotEngine(EngineParams(slots=slots, prime_bits=CHAIN))


def encode_pair(eng, a, b, extra_width: int = 0):  # test_matmul.py:12-25
    a, b = np.atleast_2d(np.asarray(a, float)), np.atleast_2d(np.asarray(b, float))
    m, n = a.shape
    p = b.shape[1]
    width = max(n, p) + extra_width
    ap = np.zeros((m, width))
    ap[:, :n] = a
    bp = np.zeros((width, p))
    bp[:n] = b
    return encode_row_major(eng, ap), encode_revolver(eng, bp, target_m=max(m, p))


def meter(d):
    return [d.add_count, d.mul_count, d.cmul_count, d.rot_count, d.enc_count, d.max_depth]


def test_row_shifter_paths(rng):  # test_matmul.py:28-64
    eng = make_engine(8)
    bbar = encode_revolver(eng, np.array([[1, 2], [3, 4], [5, 6], [7, 8]], dtype=float), target_m=2)
    np.testing.assert_allclose(row_shifter(eng, bbar, p=2, idx=0).decode(eng), [[2, 4, 6, 8], [1, 3, 5, 7]], atol=TOL)
    eng = make_engine(16)
    bbar = encode_revolver(eng, rand_int_matrix(rng, 4, 2), target_m=4)
    before = eng.meter_snapshot()
    out = row_shifter(eng, bbar, p=2, idx=0)
    d = eng.meter_snapshot().delta_since(before)
    assert (d.rot_count, d.cmul_count, d.add_count) == (1, 0, 0)
    np.testing.assert_allclose(eng.dec(out.ct), np.roll(eng.dec(bbar.ct), -4), atol=TOL)
    eng = make_engine(64)
    bbar = encode_revolver(eng, rand_int_matrix(rng, 4, 3), target_m=3)
    before = eng.meter_snapshot()
    row_shifter(eng, bbar, p=3, idx=1)
    d = eng.meter_snapshot().delta_since(before)
    assert (d.rot_count, d.cmul_count, d.add_count) == (2, 2, 1)
    eng = make_engine(32)
    bbar = encode_revolver(eng, rand_int_matrix(rng, 4, 1), target_m=3)
    np.testing.assert_allclose(row_shifter(eng, bbar, p=1, idx=0).decode(eng), bbar.decode(eng), atol=TOL)
    with pytest.raises(EngineError):
        row_shifter(eng, bbar, p=1, idx=1)


def test_selector_and_zero_operand():  # test_matmul.py:78-91
    eng = make_engine(8)
    a = np.array([[1, 0, 0, 0], [0, 1, 0, 0]], dtype=float)
    b = np.array([[1, 2], [3, 4], [5, 6], [7, 8]], dtype=float)
    np.testing.assert_allclose(matmul(eng, *encode_pair(eng, a, b)).decode(eng)[:2, :2], [[1, 2], [3, 4]], atol=TOL)
    got = matmul(eng, *encode_pair(eng, np.zeros((2, 4)), np.arange(8, dtype=float).reshape(4, 2))).decode(eng)
    assert np.abs(got).max() < TOL


@pytest.mark.parametrize("extra", [1, 4], ids=["full-pack", "slack-slots"])
def test_oracle_grid(rng, extra):  # test_matmul.py:94-109
    engines = {}
    for m in (1, 2, 4, 8):
        for n in (1, 2, 4, 8):
            for p in (1, 2, 4, 8):
                slots = max(2, max(m, p) * max(n, p) * extra)
                eng = engines.setdefault(slots, make_engine(slots))
                a, b = rand_int_matrix(rng, m, n), rand_int_matrix(rng, n, p)
                got = matmul(eng, *encode_pair(eng, a, b)).decode(eng)
                np.testing.assert_allclose(got[:m, :p], a @ b, atol=TOL)
                got[:m, :p] = 0
                assert np.abs(got).max() < TOL


def test_non_pow2_rows_and_bias(rng):  # test_matmul.py:112-118, 173-184
    eng = make_engine(64)
    a, b = rand_int_matrix(rng, 3, 4), rand_int_matrix(rng, 4, 2)
    np.testing.assert_allclose(matmul(eng, *encode_pair(eng, a, b)).decode(eng)[:3, :2], a @ b, atol=TOL)
    eng = make_engine(16)
    a, b = rand_int_matrix(rng, 4, 4), rand_int_matrix(rng, 4, 2)
    seed = np.zeros((4, 4))
    seed[:, :2] = [10.0, 20.0]
    got = matmul(eng, *encode_pair(eng, a, b), init=eng.enc(seed.reshape(-1))).decode(eng)
    np.testing.assert_allclose(got[:4, :2], a @ b + np.array([10.0, 20.0]), atol=TOL)


def test_costs_and_depth(rng):  # test_matmul.py:121-170
    m = n = p = 4
    eng = make_engine(16)
    ca, cb = encode_pair(eng, rand_int_matrix(rng, m, n), rand_int_matrix(rng, n, p))
    before = eng.meter_snapshot()
    out = matmul(eng, ca, cb)
    d = eng.meter_snapshot().delta_since(before)
    assert d.rot_count == p * (1 + 2 * (n.bit_length() - 1)) and d.mul_count == p
    assert out.ct.depth == 3
    m, n, p = 3, 4, 2
    eng = make_engine(32)
    ca, cb = encode_pair(eng, rand_int_matrix(rng, m, n), rand_int_matrix(rng, n, p))
    before = eng.meter_snapshot()
    matmul(eng, ca, cb)
    d = eng.meter_snapshot().delta_since(before)
    assert d.rot_count == p * (2 + 2 * (n.bit_length() - 1)) and d.cmul_count == p * 4
    for p in (2, 4, 8):
        eng = make_engine(256)
        ca, cb = encode_pair(eng, rand_int_matrix(rng, 8, 8), rand_int_matrix(rng, 8, p))
        assert matmul(eng, ca, cb).ct.depth == 4
    assert not MatmulPlan.plan(make_engine(32), 4, 4, 2).fast_path


def test_tiled(rng):  # test_matmul.py:187-215
    eng = make_engine(16)
    a, b = rand_int_matrix(rng, 8, 4), rand_int_matrix(rng, 4, 2)
    tops, bots = encode_pair(eng, a[:4], b), encode_pair(eng, a[4:], b)
    out = matmul_tiled(eng, [tops[0], bots[0]], [tops[1]])
    np.testing.assert_allclose(np.vstack([out[0].decode(eng)[:4, :2], out[1].decode(eng)[:4, :2]]), a @ b, atol=TOL)
    a, b = rand_int_matrix(rng, 4, 4), rand_int_matrix(rng, 4, 4)
    ca, cl = encode_pair(eng, a, b[:, :2])
    _, cr = encode_pair(eng, a, b[:, 2:])
    out = matmul_tiled(eng, [ca], [cl, cr])
    np.testing.assert_allclose(np.hstack([out[0].decode(eng)[:4, :2], out[1].decode(eng)[:4, :2]]), a @ b, atol=TOL)
    with pytest.raises(LayoutError):
        matmul_tiled(eng, [ca], [], grid=(1, 0))


@pytest.mark.parametrize("idx", range(8))
def test_reference_fixtures(golden, idx):
    """Decoded values, meter deltas and depth equal the reference's own run (make_golden.py a3_*)."""
    m, n, p, slots = (int(x) for x in golden[f"a3_{idx}_shape"])
    eng = make_engine(slots)
    ca, cb = encode_pair(eng, golden[f"a3_{idx}_a"], golden[f"a3_{idx}_b"])
    before = eng.meter_snapshot()
    out = matmul(eng, ca, cb)
    d = eng.meter_snapshot().delta_since(before)
    assert meter(d)[:5] == list(golden[f"a3_{idx}_meter"][:5])
    assert out.ct.depth == int(golden[f"a3_{idx}_depth"][0])
    np.testing.assert_allclose(out.decode(eng), golden[f"a3_{idx}_out"], atol=TOL)


@pytest.mark.parametrize("idx", [0, 1, 4, 6])
def test_residues_bit_exact_vs_oracle(golden, idx):
    """Batched GPU Alg 3 == per-iteration Alg 3 on the C oracle, residue for residue."""
    m, n, p, slots = (int(x) for x in golden[f"a3_{idx}_shape"])
    a, b = golden[f"a3_{idx}_a"], golden[f"a3_{idx}_b"]
    eng = make_engine(slots)
    gpu = matmul(eng, *encode_pair(eng, a, b))
    orc = OracleEngine(slots, CHAIN, seed=0)
    ref = matmul(orc, *encode_pair(orc, a, b))
    assert gpu.ct.level == ref.ct.level
    np.testing.assert_array_equal(gpu.ct.residues(), ref.ct.data)
    # and the GPU's own per-iteration loop gives the same residues as its batched path
    eng2 = make_engine(slots)
    loop = matmul(eng2, *encode_pair(eng2, a, b), batched=False)
    np.testing.assert_array_equal(loop.ct.residues(), ref.ct.data)


def test_cfg2_alg3_full_width():
    """BASELINE config 2's "exercises rotations" reading: A, B 64x64 padded to width 128 so the
    64x128 layout fills the 8192 slots (fast path, depth 3), on the cfg-2 chain."""
    from paper_2512_18646_b200 import config_params

    r = np.random.default_rng(1)
    a, b = r.uniform(-1, 1, (64, 64)), r.uniform(-1, 1, (64, 64))
    eng = SlotEngine(config_params(2))
    ca, cb = encode_pair(eng, a, b, extra_width=64)
    assert MatmulPlan.plan(eng, 64, 128, 64).fast_path
    out = matmul(eng, ca, cb)
    assert out.ct.depth == 3
    got = out.decode(eng)
    assert np.abs(got[:, :64] - a @ b).max() < TOL
    assert np.abs(got[:, 64:]).max() < TOL
