"""Drop-in proof: the reference's own op sequences, driven one engine call at a
time, run unchanged on the GPU engine.

oracle/sim.py restates the reference loops line by line against the SlotEngine
surface -- matmul_outer (multicipher.py:88-103), encode_image_columns /
conv_columns / reassemble_columns (multicipher.py:106-172) and poly_activation
(pipeline.py:180-197).  Here they drive CkksEngine directly (per-op enc / mul /
add / cmul / rot / mask calls, no batched product drivers):

* decoded values match the fixtures the reference itself produced (<= 1e-3);
* the meter deltas (add, mul, cmul, rot, enc, max depth) and the result depth equal
  the reference's exactly;
* the same loops driven on the CPU residue oracle give bit-identical residues, so
  every per-op primitive of the chain matches the oracle, not only the batched drivers.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import sim  # noqa: E402
from oracle.engine import OracleEngine  # noqa: E402
from paper_2512_18646_b200 import EngineParams, SlotEngine  # noqa: E402

TOL = 1e-3
CHAIN = (60, 45, 45, 45, 45)


def engines(slots):
    p = EngineParams(slots=slots, prime_bits=CHAIN)
    return SlotEngine(p), OracleEngine.from_params(p)


def meter(d):
    return (d.add_count, d.mul_count, d.cmul_count, d.rot_count, d.enc_count, d.max_depth)


def test_reference_matmul_outer_loop(golden):
    for idx in range(7):
        a, b = golden[f"mm{idx}_a"], golden[f"mm{idx}_b"]
        m, p = a.shape[0], b.shape[1]
        eng, orc = engines(max(2, 1 << (m * p - 1).bit_length()))
        left, right = sim.encode_left(eng, a, p), sim.encode_right(eng, b, m)
        before = eng.meter_snapshot()
        c, acc = sim.matmul_outer(eng, left, right, m, p)
        d = eng.meter_snapshot().delta_since(before)
        np.testing.assert_allclose(c, golden[f"mm{idx}_c"], atol=TOL)
        assert meter(d) == tuple(golden[f"mm{idx}_meter"])
        assert acc.depth == int(golden[f"mm{idx}_depth"][0])
        _, oacc = sim.matmul_outer(orc, sim.encode_left(orc, a, p), sim.encode_right(orc, b, m), m, p)
        np.testing.assert_array_equal(acc.residues(), oacc.data)


def test_reference_conv_columns_loop(golden):
    for idx in range(5):
        imgs, w, bias = golden[f"cv{idx}_img"], golden[f"cv{idx}_w"], float(golden[f"cv{idx}_bias"][0])
        m, h, _ = imgs.shape
        eng, orc = engines(max(2, 1 << (m * h - 1).bit_length()))
        cts, geom = sim.encode_image_columns(eng, imgs)
        before = eng.meter_snapshot()
        out, g2 = sim.conv_columns(eng, cts, geom, w, bias)
        d = eng.meter_snapshot().delta_since(before)
        np.testing.assert_allclose(sim.reassemble_columns(eng, out, g2), golden[f"cv{idx}_out"], atol=TOL)
        assert meter(d) == tuple(golden[f"cv{idx}_meter"])
        octs, ogeom = sim.encode_image_columns(orc, imgs)
        oout, _ = sim.conv_columns(orc, octs, ogeom, w, bias)
        for gc, oc in zip(out, oout):
            np.testing.assert_array_equal(gc.residues(), oc.data)


def test_reference_poly_activation_loop(golden):
    for idx in range(4):
        x, coeffs = golden[f"pa{idx}_x"], golden[f"pa{idx}_coeffs"]
        eng, orc = engines(16)
        ct = eng.enc(x)
        before = eng.meter_snapshot()
        out = sim.poly_activation(eng, ct, coeffs)
        d = eng.meter_snapshot().delta_since(before)
        np.testing.assert_allclose(eng.dec(out), golden[f"pa{idx}_out"], atol=TOL)
        assert meter(d) == tuple(golden[f"pa{idx}_meter"])
        assert out.depth == int(golden[f"pa{idx}_depth"][0])
        oout = sim.poly_activation(orc, orc.enc(x), coeffs)
        np.testing.assert_array_equal(out.residues(), oout.data)
