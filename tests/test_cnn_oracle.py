"""conv.py / virtual.py / pipeline.py through the C residue oracle on the
CPU: the per-iteration algorithms of the package, on small shapes, decoded against fixtures
produced by the reference itself (tests/golden/make_golden.py cs*/bc/rf/vr/fc*)."""

import numpy as np
import pytest

from oracle.engine import OracleEngine
from oracle.sim import oracle_conv, oracle_flatten
from paper_2512_18646_b200.conv import ImageShape, Kernel, conv, kernel_spanner, span_matrix
from paper_2512_18646_b200.encoding import encode_db
from paper_2512_18646_b200.errors import EngineError, LayoutError
from paper_2512_18646_b200.pipeline import BatchPlan, ModelWeights, _fc_blocking, fc_layer, pack_batch
from paper_2512_18646_b200.virtual import VirtualLayout, batched_conv, reform, tile_kernel_span, vrot

TOL = 1e-3
CHAIN = (60, 45, 45, 45, 45)


def oracle(slots):
    return OracleEngine(slots, CHAIN, seed=0)


def test_span_matrix_patterns():  # test_conv.py:27-51 (4x4 image, k = 2)
    k = Kernel(np.array([[1.0, 2.0], [3.0, 4.0]]))
    shape = ImageShape(4, 4)
    np.testing.assert_array_equal(span_matrix(k, shape, 0, 0),
                                  [[1, 2, 1, 2], [3, 4, 3, 4], [1, 2, 1, 2], [3, 4, 3, 4]])
    np.testing.assert_array_equal(span_matrix(k, shape, 1, 0),
                                  [[0, 1, 2, 0], [0, 3, 4, 0], [0, 1, 2, 0], [0, 3, 4, 0]])
    np.testing.assert_array_equal(span_matrix(k, shape, 1, 1),
                                  [[0, 0, 0, 0], [0, 1, 2, 0], [0, 3, 4, 0], [0, 0, 0, 0]])


def test_layout_and_plan_validation():  # test_virtual.py:27-34, test_pipeline.py:79-90
    with pytest.raises(EngineError):
        VirtualLayout(2, 12, 3, 4)
    with pytest.raises(EngineError):
        VirtualLayout(2, 8, 3, 3)
    lay = VirtualLayout(2, 16, 3, 4)
    assert lay.pad == 4 and lay.image_slots == 12
    plan = BatchPlan.for_dataset(10000)
    assert (plan.images_per_ct, plan.batch_count, plan.zero_fill) == (32, 313, 16)
    with pytest.raises(EngineError):
        BatchPlan.for_dataset(10, slots=100, image_slots=32)
    assert _fc_blocking(32, 64) == (32, 2) and _fc_blocking(32, 10) == (16, 1)
    with pytest.raises(LayoutError):
        _fc_blocking(12, 64)


def test_model_weights_validation():  # test_pipeline.py:206-219
    kern = [Kernel(np.zeros((3, 3))) for _ in range(4)]
    good = ModelWeights(kern, np.zeros((64, 2704)), np.zeros(64), np.zeros((10, 64)), np.zeros(10), (0,) * 4, (0,) * 4)
    good.validate()
    with pytest.raises(EngineError):
        ModelWeights(kern, np.zeros((64, 100)), np.zeros(64), np.zeros((10, 64)), np.zeros(10), (0,) * 4,
                     (0,) * 4).validate()
    with pytest.raises(EngineError):
        ModelWeights(kern[:3], np.zeros((64, 2704)), np.zeros(64), np.zeros((10, 64)), np.zeros(10), (0,) * 4,
                     (0,) * 4).validate()


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_conv_oracle_matches_reference(golden, idx):
    img, kw, bias = golden[f"cs{idx}_img"], golden[f"cs{idx}_w"], float(golden[f"cs{idx}_bias"][0])
    h, w = img.shape
    eng = oracle(max(2, 1 << (h * w - 1).bit_length()))
    shape = ImageShape(h, w)
    out = conv(eng, eng.enc(img.reshape(-1)), kernel_spanner(eng, Kernel(kw, bias=bias), shape), shape)
    assert out.depth == int(golden[f"cs{idx}_depth"][0])
    got = eng.dec(out)[: h * w].reshape(h, w)
    np.testing.assert_allclose(got, golden[f"cs{idx}_out"], atol=TOL)
    oh, ow = shape.out(kw.shape[0])
    np.testing.assert_allclose(got[:oh, :ow], oracle_conv(img, kw, bias), atol=TOL)


def test_batched_conv_reform_vrot_oracle(golden):
    lay = VirtualLayout(4, 128, 8, 8)
    eng = oracle(512)
    imgs = golden["bc_imgs"]
    ct = pack_batch(eng, imgs, lay)
    span = tile_kernel_span(eng, Kernel(golden["bc_w"], bias=0.25), lay)
    out = batched_conv(eng, ct, lay, span)
    got = eng.dec(out)
    np.testing.assert_allclose(got, golden["bc_out"], atol=TOL)
    for b in range(4):
        np.testing.assert_allclose(got.reshape(4, 128)[b, :64].reshape(8, 8)[:6, :6],
                                   oracle_conv(imgs[b], golden["bc_w"], 0.25), atol=TOL)
    flat, new = reform(eng, out, lay, 6, 6)
    assert (new.h, new.w) == (6, 6)
    rf = eng.dec(flat)
    np.testing.assert_allclose(rf, golden["rf_out"], atol=TOL)
    for b in range(4):
        np.testing.assert_allclose(rf.reshape(4, 128)[b, :36],
                                   oracle_flatten([oracle_conv(imgs[b], golden["bc_w"], 0.25)]), atol=TOL)
    np.testing.assert_allclose(eng.dec(vrot(eng, ct, lay, 5)), golden["vr_out"], atol=TOL)


@pytest.mark.parametrize("idx", [0, 1])
def test_fc_layer_oracle(golden, idx):
    x, w, b = golden[f"fc{idx}_x"], golden[f"fc{idx}_w"], golden[f"fc{idx}_b"]
    eng = oracle(32 if idx == 0 else 64)
    out = fc_layer(eng, encode_db(eng, x), w, b)
    assert out.ct.depth == int(golden[f"fc{idx}_depth"][0])
    got = out.decode(eng)
    np.testing.assert_allclose(got, golden[f"fc{idx}_out"], atol=TOL)
    np.testing.assert_allclose(got[:, : w.shape[0]], x @ w.T + b, atol=TOL)
