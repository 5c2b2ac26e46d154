"""Algorithm 3 (revolver matmul, matmul.py of the reference) on the CPU.

* host logic of paper_2512_18646_b200.matmul (plans, filters, validation) against a
  minimal slot-engine stub, mirroring test_matmul.py's non-arithmetic cases;
* the per-iteration algorithm run through the C residue oracle (OracleEngine), decoded
  against fixtures produced by the reference itself (tests/golden, make_golden.py a3_*).
"""

import numpy as np
import pytest

from oracle.engine import OracleEngine
from paper_2512_18646_b200.encoding import Encoding, MatrixShape, PackedMatrix, encode_revolver, encode_row_major
from paper_2512_18646_b200.engine import PlainMask
from paper_2512_18646_b200.errors import EngineError, LayoutError
from paper_2512_18646_b200.matmul import MatmulPlan, build_result_filter, matmul, matmul_tiled, row_shifter

TOL = 1e-3


class StubEngine:
    """Slot count + mask only: enough for the planning / filter / validation logic."""

    def __init__(self, slots):
        self.slots = slots

    def mask(self, values, role="constant"):
        full = np.zeros(self.slots)
        v = np.asarray(values, dtype=np.float64).reshape(-1)
        full[: v.size] = v
        return PlainMask(full, role=role)


def test_result_filter_placement():  # test_matmul.py:65-75
    f = build_result_filter(StubEngine(8), 2, 4, 2, 0)
    np.testing.assert_array_equal(f.values[:8].reshape(2, 4), [[1, 0, 0, 0], [0, 1, 0, 0]])
    f = build_result_filter(StubEngine(8), 2, 4, 2, 1)
    np.testing.assert_array_equal(f.values[:8].reshape(2, 4), [[0, 1, 0, 0], [1, 0, 0, 0]])
    f = build_result_filter(StubEngine(16), 3, 4, 1, 0)
    np.testing.assert_array_equal(f.values[:12].reshape(3, 4)[:, 0], [1, 1, 1])
    with pytest.raises(EngineError):
        build_result_filter(StubEngine(8), 2, 4, 2, 2)


def test_plan_fast_requires_full_pack():  # test_matmul.py:166-171
    assert not MatmulPlan.plan(StubEngine(32), 4, 4, 2).fast_path
    assert MatmulPlan.plan(StubEngine(16), 4, 4, 2).fast_path
    assert not MatmulPlan.plan(StubEngine(16), 3, 4, 2).fast_path
    with pytest.raises(LayoutError):
        MatmulPlan.plan(StubEngine(64), m=2, n=2, p=4)
    with pytest.raises(LayoutError):
        MatmulPlan.plan(StubEngine(8), m=4, n=4, p=4)


def test_validation_errors():  # test_matmul.py:146-163, 205-212
    eng = StubEngine(64)
    ct = object()
    a = PackedMatrix(ct, MatrixShape(2, 4), Encoding.ROW_MAJOR)
    b_wrong_width = PackedMatrix(ct, MatrixShape(2, 8), Encoding.REVOLVER, revolve_p=2)
    with pytest.raises(LayoutError):
        matmul(eng, a, b_wrong_width)
    with pytest.raises(LayoutError):
        matmul(eng, PackedMatrix(ct, MatrixShape(2, 4), Encoding.REVOLVER, revolve_p=2), a)
    with pytest.raises(LayoutError):
        matmul(eng, a, PackedMatrix(ct, MatrixShape(2, 4), Encoding.ROW_MAJOR))
    with pytest.raises(LayoutError):
        matmul_tiled(eng, [a], [b_wrong_width])
    with pytest.raises(LayoutError):
        matmul_tiled(eng, [a], [], grid=(1, 0))
    with pytest.raises(LayoutError):
        matmul_tiled(eng, [a], [PackedMatrix(ct, MatrixShape(2, 4), Encoding.REVOLVER, revolve_p=2)], grid=(2, 1))
    bbar = PackedMatrix(ct, MatrixShape(2, 4), Encoding.REVOLVER, revolve_p=2)
    with pytest.raises(EngineError):
        row_shifter(eng, bbar, p=2, idx=2)
    with pytest.raises(EngineError):
        row_shifter(eng, bbar, p=3, idx=0)
    with pytest.raises(LayoutError):
        row_shifter(eng, a, p=2, idx=0)


def _oracle(slots):
    return OracleEngine(slots, (60, 45, 45, 45, 45), seed=0)


def _encode_pair(eng, a, b):
    m, n = a.shape
    p = b.shape[1]
    width = max(n, p)
    ap = np.zeros((m, width))
    ap[:, :n] = a
    bp = np.zeros((width, p))
    bp[:n] = b
    return encode_row_major(eng, ap), encode_revolver(eng, bp, target_m=max(m, p))


def test_row_shifter_single_step_oracle():  # test_matmul.py:28-33
    eng = _oracle(8)
    bbar = encode_revolver(eng, np.array([[1, 2], [3, 4], [5, 6], [7, 8]], dtype=float), target_m=2)
    out = row_shifter(eng, bbar, p=2, idx=0)
    np.testing.assert_allclose(out.decode(eng), [[2, 4, 6, 8], [1, 3, 5, 7]], atol=TOL)


@pytest.mark.parametrize("idx", range(7))
def test_alg3_oracle_matches_reference(golden, idx):
    m, n, p, slots = (int(x) for x in golden[f"a3_{idx}_shape"])
    a, b = golden[f"a3_{idx}_a"], golden[f"a3_{idx}_b"]
    eng = _oracle(slots)
    ca, cb = _encode_pair(eng, a, b)
    out = matmul(eng, ca, cb)
    assert out.ct.depth == int(golden[f"a3_{idx}_depth"][0])
    got = out.decode(eng)
    np.testing.assert_allclose(got, golden[f"a3_{idx}_out"], atol=TOL)
    np.testing.assert_allclose(got[:m, :p], a @ b, atol=TOL)
