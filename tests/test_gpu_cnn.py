"""conv.py / virtual.py / pipeline.py (the dataset-layout CNN of the paper's Table 1) on the GPU
engine: the reference's test_conv / test_virtual / test_pipeline cases (exact equality ->
<= 1e-3 decoded error, meters and depths exact), bit-exact residues of the batched GPU paths
against the per-iteration algorithms on the C residue oracle, and the full 32-image forward pass
at the paper's layout against the reference's own scores and stage meters."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.engine import OracleEngine  # noqa: E402
from oracle.sim import oracle_conv, oracle_flatten, oracle_forward, table1_weights  # noqa: E402
from paper_2512_18646_b200 import (  # noqa: E402
    PIPELINE_DEPTH, EngineError, EngineParams, ImageShape, Kernel, LayoutError, ModelWeights, SlotEngine,
    VirtualLayout, argmax_decide, batched_conv, build_offset_filter, conv, encode_db, encode_model, fc_layer,
    flatten_maps, forward_encoded, kernel_spanner, pack_batch, reform, sum_for_conv, tile_kernel_span, vadd, vmul,
    vrot)
from paper_2512_18646_b200.pipeline import conv_layer  # noqa: E402

from conftest import rand_int_matrix  # noqa: E402

TOL = 1e-3
CHAIN = (60, 45, 45, 45, 45)
ACT1 = (-0.00015120704, 0.4610149, 2.0225089, -1.4511951)
ACT2 = (-1.5650465, -0.9943767, 1.6794522, 0.5350255)


def make_engine(slots):
    return SlotEngine(EngineParams(slots=slots, prime_bits=CHAIN))


def meter(d):
    return [d.add_count, d.mul_count, d.cmul_count, d.rot_count, d.enc_count]


@pytest.mark.parametrize("idx", range(4))
def test_conv_reference_fixtures(golden, idx):  # test_conv.py:152-191 shapes
    img, kw, bias = golden[f"cs{idx}_img"], golden[f"cs{idx}_w"], float(golden[f"cs{idx}_bias"][0])
    h, w = img.shape
    eng = make_engine(max(2, 1 << (h * w - 1).bit_length()))
    shape = ImageShape(h, w)
    span = kernel_spanner(eng, Kernel(kw, bias=bias), shape)
    ct = eng.enc(img.reshape(-1))
    before = eng.meter_snapshot()
    out = conv(eng, ct, span, shape)
    d = eng.meter_snapshot().delta_since(before)
    assert meter(d) == list(golden[f"cs{idx}_meter"][:5])
    assert out.depth == int(golden[f"cs{idx}_depth"][0])
    got = eng.dec(out)[: h * w].reshape(h, w)
    np.testing.assert_allclose(got, golden[f"cs{idx}_out"], atol=TOL)


def test_sum_for_conv_and_filters(rng):  # test_conv.py:75-150
    eng = make_engine(16)
    shape = ImageShape(4, 4)
    out = eng.dec(sum_for_conv(eng, eng.enc(np.ones(16)), shape, 2)).reshape(4, 4)
    np.testing.assert_allclose(out, [[4, 0, 4, 0], [0, 0, 0, 0], [4, 0, 4, 0], [0, 0, 0, 0]], atol=TOL)
    img = rand_int_matrix(rng, 4, 4)
    before = eng.meter_snapshot()
    out = eng.dec(sum_for_conv(eng, eng.enc(img.reshape(-1)), shape, 2, bias=1.5)).reshape(4, 4)
    assert eng.meter_snapshot().delta_since(before).rot_count == 4
    for y in (0, 2):
        for x in (0, 2):
            assert abs(out[y, x] - (img[y:y + 2, x:x + 2].sum() + 1.5)) < TOL
    eng6 = make_engine(64)
    s6 = ImageShape(6, 6)
    total = sum(build_offset_filter(eng6, s6, 3, i, j).values[:36].reshape(6, 6) for i in range(3) for j in range(3))
    valid = np.zeros((6, 6))
    valid[:4, :4] = 1
    np.testing.assert_array_equal(total, valid)
    with pytest.raises(EngineError):
        build_offset_filter(eng6, s6, 3, 3, 0)
    with pytest.raises(EngineError):
        kernel_spanner(eng6, Kernel(np.ones((3, 3))), ImageShape(4, 6))


def test_virtual_ops(rng):  # test_virtual.py:36-98
    eng = make_engine(32)
    lay = VirtualLayout(2, 16, 3, 4)
    rows = np.array([np.arange(1, 13), np.arange(13, 25)], dtype=float)
    ct = pack_batch(eng, rows.reshape(2, 3, 4), lay)
    out = eng.dec(vrot(eng, ct, lay, 4)).reshape(2, 16)
    for b in range(2):
        np.testing.assert_allclose(out[b, :12], np.roll(rows[b], -4), atol=TOL)
    assert np.abs(out[:, 12:]).max() < TOL
    np.testing.assert_allclose(eng.dec(vrot(eng, ct, lay, 0)).reshape(2, 16)[:, :12], rows, atol=TOL)
    with pytest.raises(EngineError):
        vrot(eng, ct, lay, 12)
    a = pack_batch(eng, rand_int_matrix(rng, 2, 12).reshape(2, 3, 4), lay)
    np.testing.assert_allclose(eng.dec(vadd(eng, a, ct)), eng.dec(a) + eng.dec(ct), atol=TOL)
    np.testing.assert_allclose(eng.dec(vmul(eng, a, ct)), eng.dec(a) * eng.dec(ct), atol=5e-3)
    other = eng.enc(np.ones(32), layout=("dataset", 4, 8, 2, 4))
    with pytest.raises(LayoutError):
        vadd(eng, ct, other)


def test_batched_conv_reform_fixtures(golden):  # test_virtual.py:100-183
    lay = VirtualLayout(4, 128, 8, 8)
    eng = make_engine(512)
    ct = pack_batch(eng, golden["bc_imgs"], lay)
    span = tile_kernel_span(eng, Kernel(golden["bc_w"], bias=0.25), lay)
    before = eng.meter_snapshot()
    out = batched_conv(eng, ct, lay, span)
    assert meter(eng.meter_snapshot().delta_since(before)) == list(golden["bc_meter"][:5])
    np.testing.assert_allclose(eng.dec(out), golden["bc_out"], atol=TOL)
    before = eng.meter_snapshot()
    flat, _ = reform(eng, out, lay, 6, 6)
    assert meter(eng.meter_snapshot().delta_since(before)) == list(golden["rf_meter"][:5])
    np.testing.assert_allclose(eng.dec(flat), golden["rf_out"], atol=TOL)
    before = eng.meter_snapshot()
    np.testing.assert_allclose(eng.dec(vrot(eng, ct, lay, 5)), golden["vr_out"], atol=TOL)
    assert meter(eng.meter_snapshot().delta_since(before)) == list(golden["vr_meter"][:5])
    with pytest.raises(LayoutError):
        batched_conv(eng, ct, VirtualLayout(4, 128, 8, 8), tile_kernel_span(eng, Kernel(np.ones((3, 3))),
                                                                            VirtualLayout(4, 128, 7, 8)))
    tight = VirtualLayout(8, 64, 7, 8)
    with pytest.raises(LayoutError):
        batched_conv(eng, ct, tight, tile_kernel_span(eng, Kernel(np.ones((3, 3))), tight))
    with pytest.raises(EngineError):
        reform(eng, out, lay, 9, 6)


def test_conv_layer_and_flatten(rng):  # test_pipeline.py:106-153
    eng = make_engine(512)
    lay = VirtualLayout(4, 128, 8, 8)
    spans = [tile_kernel_span(eng, Kernel(np.zeros((3, 3)), bias=b), lay) for b in (1.0, -2.0)]
    outs, _, (oh, ow) = conv_layer(eng, pack_batch(eng, rng.uniform(0, 1, size=(4, 8, 8)), lay), lay, spans)
    assert (oh, ow) == (6, 6)
    for out, bias in zip(outs, (1.0, -2.0)):
        grid = eng.dec(out).reshape(4, 128)[:, :64].reshape(4, 8, 8)
        np.testing.assert_allclose(grid[:, :6, :6], np.full((4, 6, 6), bias), atol=TOL)
    maps = rng.integers(-3, 9, size=(2, 4, 6, 6)).astype(float)
    cts = []
    for c in range(2):
        grid = np.full((4, 128), 7.5)
        for b in range(4):
            img = np.zeros((8, 8))
            img[:6, :6] = maps[c, b]
            grid[b, :64] = img.reshape(-1)
        cts.append(eng.enc(grid.reshape(-1)))
    data = flatten_maps(eng, cts, lay, 6, 6)
    assert data.valid_widths == [36, 36]
    for b in range(4):
        got = np.concatenate([ch.decode(eng)[b, :36] for ch in data.chunks])
        np.testing.assert_allclose(got, oracle_flatten([maps[0, b], maps[1, b]]), atol=TOL)
        for ch in data.chunks:
            assert np.abs(ch.decode(eng)[b, 36:]).max() < TOL


@pytest.mark.parametrize("idx", [0, 1])
def test_fc_layer_fixtures(golden, idx):  # test_pipeline.py:156-203
    x, w, b = golden[f"fc{idx}_x"], golden[f"fc{idx}_w"], golden[f"fc{idx}_b"]
    eng = make_engine(32 if idx == 0 else 64)
    pm = encode_db(eng, x)
    before = eng.meter_snapshot()
    out = fc_layer(eng, pm, w, b)
    assert meter(eng.meter_snapshot().delta_since(before)) == list(golden[f"fc{idx}_meter"][:5])
    assert out.ct.depth == int(golden[f"fc{idx}_depth"][0])
    np.testing.assert_allclose(out.decode(eng), golden[f"fc{idx}_out"], atol=TOL)
    with pytest.raises(LayoutError):
        fc_layer(eng, pm, np.ones((4, x.shape[1])), np.ones(3))


def test_residues_bit_exact_vs_oracle(golden):
    """Batched GPU conv / batched_conv / reform / fc_layer == the per-iteration algorithms on the
    C residue oracle, residue for residue."""
    img, kw = golden["cs1_img"], golden["cs1_w"]
    shape = ImageShape(*img.shape)
    for eng in (make_engine(64), OracleEngine(64, CHAIN, seed=0)):
        out = conv(eng, eng.enc(img.reshape(-1)), kernel_spanner(eng, Kernel(kw, bias=0.5), shape), shape)
        res = out.residues() if hasattr(out, "residues") else out.data
        if isinstance(eng, OracleEngine):
            np.testing.assert_array_equal(gpu_res, res)
        else:
            gpu_res = res
    lay = VirtualLayout(4, 128, 8, 8)
    outs = []
    for eng in (make_engine(512), OracleEngine(512, CHAIN, seed=0)):
        ct = pack_batch(eng, golden["bc_imgs"], lay)
        bc = batched_conv(eng, ct, lay, tile_kernel_span(eng, Kernel(golden["bc_w"], bias=0.25), lay))
        flat, _ = reform(eng, bc, lay, 6, 6)
        outs.append(flat.residues() if hasattr(flat, "residues") else flat.data)
    np.testing.assert_array_equal(outs[0], outs[1])
    outs = []
    for eng in (make_engine(64), OracleEngine(64, CHAIN, seed=0)):
        r = fc_layer(eng, encode_db(eng, golden["fc1_x"]), golden["fc1_w"], golden["fc1_b"])
        outs.append(r.ct.residues() if hasattr(r.ct, "residues") else r.ct.data)
    np.testing.assert_array_equal(outs[0], outs[1])


def _table1_weights(seed):
    kw, kb, f1w, f1b, f2w, f2b = table1_weights(seed)
    return ModelWeights([Kernel(kw[i], bias=float(kb[i])) for i in range(4)], f1w, f1b, f2w, f2b, ACT1, ACT2)


def test_table1_forward_matches_reference(golden):
    """The paper's encrypted CNN: 32 images of 28x28 in one 32768-slot ciphertext, depth 13, on a
    14-prime chain (q0 60b + 13 x 45b + P 60b), N = 2^16."""
    eng = SlotEngine(EngineParams(slots=32768, prime_bits=(60,) + (45,) * 13))
    weights = _table1_weights(7)
    imgs = np.random.default_rng(8).uniform(0, 1, size=(32, 28, 28))
    model = encode_model(eng, weights)
    assert model.ciphertext_count == int(golden["t1_depth"][1]) == 52
    ct = pack_batch(eng, imgs)
    sm = {}
    scores = forward_encoded(eng, ct, model, stage_meters=sm)
    got = scores.decode(eng)[:, :10]
    np.testing.assert_allclose(got, golden["t1_scores"], atol=TOL)
    np.testing.assert_allclose(got, oracle_forward(weights, imgs), atol=TOL)
    want = golden["t1_stage_meters"]
    for n, k in enumerate(("conv", "act1", "flatten", "fc1", "act2", "fc2")):
        assert meter(sm[k]) == list(want[n][:5]), k
    assert eng.meter_snapshot().max_depth == PIPELINE_DEPTH == int(golden["t1_depth"][0])
    np.testing.assert_array_equal(argmax_decide(eng, scores), np.argmax(golden["t1_scores"], axis=1))
