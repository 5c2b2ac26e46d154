"""Generate decoded-value fixtures by running the REFERENCE package itself.

Run in the build container (needs /root/reference):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
Writes tests/golden/reference_golden.npz.  Each case stores the seeded inputs,
the reference outputs and the reference meter deltas, so tests can pin
oracle/sim.py (and, on the GPU, the CKKS engine's decoded values) against the
reference without /root/reference being present.
"""

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from packedhe.conv import Kernel  # noqa: E402
from packedhe.engine import EngineParams, SlotEngine  # noqa: E402
from packedhe.multicipher import (  # noqa: E402
    conv_columns, encode_image_columns, encode_left, encode_right, matmul_outer, reassemble_columns)
from packedhe.pipeline import poly_activation  # noqa: E402

OUT = Path(__file__).resolve().parent / "reference_golden.npz"


def meter_tuple(d):
    return np.array([d.add_count, d.mul_count, d.cmul_count, d.rot_count, d.enc_count, d.max_depth])


def main():
    rng = np.random.default_rng(0xC0FFEE)
    data = {}
    # matmul_outer grid (acceptance criterion 2 shapes) + BASELINE cfg1/cfg2 shapes
    mm = [(1, 1, 1), (2, 2, 2), (2, 4, 2), (4, 8, 4), (8, 2, 2), (8, 16, 4), (3, 5, 7)]
    for idx, (m, n, p) in enumerate(mm):
        a = rng.integers(-4, 5, size=(m, n)).astype(float)
        b = rng.integers(-4, 5, size=(n, p)).astype(float)
        eng = SlotEngine(EngineParams(slots=max(2, 1 << (m * p - 1).bit_length())))
        left, right = encode_left(eng, a, p), encode_right(eng, b, m)
        before = eng.meter_snapshot()
        out = matmul_outer(eng, left, right)
        d = eng.meter_snapshot().delta_since(before)
        data[f"mm{idx}_a"], data[f"mm{idx}_b"] = a, b
        data[f"mm{idx}_c"] = out.decode(eng)
        data[f"mm{idx}_meter"] = meter_tuple(d)
        data[f"mm{idx}_depth"] = np.array([out.ct.depth])
    for cfg, (seed, dim, slots) in {1: (0, 8, 4096), 2: (1, 64, 8192)}.items():
        r = np.random.default_rng(seed)
        a = r.uniform(-1, 1, (dim, dim))
        b = r.uniform(-1, 1, (dim, dim))
        eng = SlotEngine(EngineParams(slots=slots))
        out = matmul_outer(eng, encode_left(eng, a, dim), encode_right(eng, b, dim))
        data[f"cfg{cfg}_a"], data[f"cfg{cfg}_b"], data[f"cfg{cfg}_c"] = a, b, out.decode(eng)
    # conv_columns cases
    cc = [(2, 6, 6, 3, 0.5), (1, 5, 7, 2, -1.0), (3, 8, 5, 3, 0.0), (2, 16, 16, 3, 0.5), (1, 9, 9, 5, 2.0)]
    for idx, (m, h, w, k, bias) in enumerate(cc):
        imgs = rng.integers(-2, 5, size=(m, h, w)).astype(float)
        kw = rng.integers(-4, 5, size=(k, k)).astype(float)
        kw[0, k - 1] = 0.0  # exercise the zero-tap skip
        eng = SlotEngine(EngineParams(slots=max(2, 1 << (m * h - 1).bit_length())))
        cei = encode_image_columns(eng, imgs)
        before = eng.meter_snapshot()
        out = conv_columns(eng, cei, Kernel(kw, bias=bias))
        d = eng.meter_snapshot().delta_since(before)
        data[f"cv{idx}_img"], data[f"cv{idx}_w"], data[f"cv{idx}_bias"] = imgs, kw, np.array([bias])
        data[f"cv{idx}_out"] = reassemble_columns(eng, out)
        data[f"cv{idx}_meter"] = meter_tuple(d)
    # poly_activation cases
    pc = [(0.25, 0.5, 0.125, 0.0), (-0.00015120704, 0.4610149, 2.0225089, -1.4511951),
          (-1.5650465, -0.9943767, 1.6794522, 0.5350255), (0.0, 1.0, 0.0, 0.0)]
    for idx, coeffs in enumerate(pc):
        x = rng.uniform(-1, 1, size=16)
        eng = SlotEngine(EngineParams(slots=16))
        ct = eng.enc(x)
        before = eng.meter_snapshot()
        out = poly_activation(eng, ct, coeffs)
        d = eng.meter_snapshot().delta_since(before)
        data[f"pa{idx}_x"], data[f"pa{idx}_coeffs"] = x, np.array(coeffs)
        data[f"pa{idx}_out"] = eng.dec(out)
        data[f"pa{idx}_meter"] = meter_tuple(d)
        data[f"pa{idx}_depth"] = np.array([out.depth])
    # rotation golden (test_engine.py:87-106)
    eng = SlotEngine(EngineParams(slots=8))
    x = np.arange(1, 9, dtype=float)
    ct = eng.enc(x)
    data["rot_x"] = x
    data["rot_steps"] = np.array([1, -1, 3, 8, -9])
    data["rot_out"] = np.stack([eng.dec(eng.rot(ct, s)) for s in data["rot_steps"]])
    # Algorithm 3 (revolver matmul, matmul.py) cases: (m, n, p, slots); operands padded like
    # test_matmul.py:12-25 (row width max(n, p), layout height max(m, p)).  Separate generator so
    # the fixtures above keep their draws.
    from packedhe.encoding import encode_revolver, encode_row_major
    from packedhe.matmul import matmul as alg3

    r3 = np.random.default_rng(0xA163)
    a3 = [(4, 4, 4, 16), (3, 4, 2, 32), (8, 8, 8, 64), (8, 8, 4, 256), (2, 4, 2, 8), (1, 2, 1, 8), (4, 4, 2, 16),
          (16, 16, 16, 256)]
    for idx, (m, n, p, slots) in enumerate(a3):
        if idx == len(a3) - 1:
            a, b = r3.uniform(-1, 1, (m, n)), r3.uniform(-1, 1, (n, p))
        else:
            a, b = r3.integers(-4, 5, size=(m, n)).astype(float), r3.integers(-4, 5, size=(n, p)).astype(float)
        width = max(n, p)
        ap = np.zeros((m, width))
        ap[:, :n] = a
        bp = np.zeros((width, p))
        bp[:n] = b
        eng = SlotEngine(EngineParams(slots=slots))
        ca, cb = encode_row_major(eng, ap), encode_revolver(eng, bp, target_m=max(m, p))
        before = eng.meter_snapshot()
        out = alg3(eng, ca, cb)
        d = eng.meter_snapshot().delta_since(before)
        data[f"a3_{idx}_shape"] = np.array([m, n, p, slots])
        data[f"a3_{idx}_a"], data[f"a3_{idx}_b"] = a, b
        data[f"a3_{idx}_out"] = out.decode(eng)
        data[f"a3_{idx}_meter"] = meter_tuple(d)
        data[f"a3_{idx}_depth"] = np.array([out.ct.depth])
    # conv.py / virtual.py / pipeline.py (the dataset-layout CNN); own generator
    from packedhe.conv import ImageShape, conv, kernel_spanner
    from packedhe.encoding import encode_db
    from packedhe.pipeline import ModelWeights, conv_layer, encode_model, fc_layer, flatten_maps, forward_encoded, pack_batch
    from packedhe.virtual import VirtualLayout, batched_conv, reform, tile_kernel_span, vrot

    rc = np.random.default_rng(0xC0DE)
    for idx, (h, w, k) in enumerate([(4, 4, 2), (6, 6, 3), (5, 7, 2), (8, 8, 3)]):
        img = rc.integers(-3, 5, size=(h, w)).astype(float)
        kw = rc.integers(-3, 4, size=(k, k)).astype(float)
        bias = float(rc.integers(-2, 3)) / 2
        slots = max(2, 1 << (h * w - 1).bit_length())
        eng = SlotEngine(EngineParams(slots=slots))
        span = kernel_spanner(eng, Kernel(kw, bias=bias), ImageShape(h, w))
        ct = eng.enc(img.reshape(-1))
        before = eng.meter_snapshot()
        out = conv(eng, ct, span, ImageShape(h, w))
        d = eng.meter_snapshot().delta_since(before)
        data[f"cs{idx}_img"], data[f"cs{idx}_w"], data[f"cs{idx}_bias"] = img, kw, np.array([bias])
        data[f"cs{idx}_out"] = eng.dec(out)[: h * w].reshape(h, w)
        data[f"cs{idx}_meter"] = meter_tuple(d)
        data[f"cs{idx}_depth"] = np.array([out.depth])
    # batched conv + reform + vrot on a 4 x 128 layout of 8x8 images
    lay = VirtualLayout(4, 128, 8, 8)
    imgs = rc.integers(0, 4, size=(4, 8, 8)).astype(float)
    kw = rc.integers(-3, 4, size=(3, 3)).astype(float)
    eng = SlotEngine(EngineParams(slots=512))
    ct = pack_batch(eng, imgs, lay)
    span = tile_kernel_span(eng, Kernel(kw, bias=0.25), lay)
    before = eng.meter_snapshot()
    out = batched_conv(eng, ct, lay, span)
    d = eng.meter_snapshot().delta_since(before)
    data["bc_imgs"], data["bc_w"], data["bc_out"] = imgs, kw, eng.dec(out)
    data["bc_meter"], data["bc_depth"] = meter_tuple(d), np.array([out.depth])
    before = eng.meter_snapshot()
    flat, _ = reform(eng, out, lay, 6, 6)
    d = eng.meter_snapshot().delta_since(before)
    data["rf_out"], data["rf_meter"] = eng.dec(flat), meter_tuple(d)
    before = eng.meter_snapshot()
    vr = vrot(eng, ct, lay, 5)
    d = eng.meter_snapshot().delta_since(before)
    data["vr_out"], data["vr_meter"] = eng.dec(vr), meter_tuple(d)
    # fc_layer: plain, and neuron blocks wider than the row count
    for idx, (rows, width, outs, slots) in enumerate([(4, 8, 4, 32), (4, 16, 8, 64)]):
        x = rc.integers(-4, 5, size=(rows, width)).astype(float)
        wmat = rc.uniform(-1, 1, size=(outs, width))
        b = rc.uniform(-1, 1, size=outs)
        eng = SlotEngine(EngineParams(slots=slots))
        pm = encode_db(eng, x)
        before = eng.meter_snapshot()
        out = fc_layer(eng, pm, wmat, b)
        d = eng.meter_snapshot().delta_since(before)
        data[f"fc{idx}_x"], data[f"fc{idx}_w"], data[f"fc{idx}_b"] = x, wmat, b
        data[f"fc{idx}_out"], data[f"fc{idx}_meter"] = out.decode(eng), meter_tuple(d)
        data[f"fc{idx}_depth"] = np.array([out.ct.depth])
    # Table-1 forward at the paper's layout (32 images of 28x28 per 32768 slots), seeded model
    sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
    from oracle.sim import table1_weights

    act1 = (-0.00015120704, 0.4610149, 2.0225089, -1.4511951)
    act2 = (-1.5650465, -0.9943767, 1.6794522, 0.5350255)
    kw4, kb4, f1w, f1b, f2w, f2b = table1_weights(7)
    weights = ModelWeights([Kernel(kw4[i], bias=float(kb4[i])) for i in range(4)], f1w, f1b, f2w, f2b, act1, act2)
    imgs = np.random.default_rng(8).uniform(0, 1, size=(32, 28, 28))
    eng = SlotEngine(EngineParams(slots=32768))
    model = encode_model(eng, weights)
    ct = pack_batch(eng, imgs)
    sm = {}
    scores = forward_encoded(eng, ct, model, stage_meters=sm)
    data["t1_scores"] = scores.decode(eng)[:, :10]
    data["t1_stage_meters"] = np.stack([meter_tuple(sm[k]) for k in ("conv", "act1", "flatten", "fc1", "act2", "fc2")])
    data["t1_depth"] = np.array([eng.meter_snapshot().max_depth, model.ciphertext_count])
    np.savez_compressed(OUT, **data)
    print(f"wrote {OUT} ({len(data)} arrays)")


if __name__ == "__main__":
    main()
