"""serial.py on the GPU engine (test_serial.py of the reference): real residue ciphertexts,
batches and encoded models round-trip bit-exactly and decrypt to the same values; loading does
not touch the meter and refuses incompatible engines."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2512_18646_b200 import EngineParams, Kernel, ModelWeights, SlotEngine, encode_model, pack_batch  # noqa: E402
from paper_2512_18646_b200.serial import (SerialError, load_batch, load_ciphertext, load_model,  # noqa: E402
                                          write_batch, write_ciphertext, write_model)
from paper_2512_18646_b200.virtual import VirtualLayout  # noqa: E402

TOL = 1e-3


def test_ciphertext_round_trip(tmp_path, rng):
    eng = SlotEngine(EngineParams(slots=64, prime_bits=(60, 45, 45)))
    x = rng.uniform(-1, 1, 64)
    ct = eng.mul(eng.enc(x, layout=("grid", 8, 8)), eng.enc(x))
    write_ciphertext(tmp_path / "c.vrct", ct, meta={"who": "test"}, engine=eng)
    before = eng.meter_snapshot()
    back, hdr = load_ciphertext(eng, tmp_path / "c.vrct")
    assert eng.meter_snapshot() == before
    np.testing.assert_array_equal(back.residues(), ct.residues())
    assert (back.level, back.scale, back.depth, back.layout) == (ct.level, ct.scale, ct.depth, ct.layout)
    np.testing.assert_allclose(eng.dec(back), x * x, atol=TOL)
    np.testing.assert_allclose(eng.dec(eng.add(back, ct)), 2 * x * x, atol=TOL)
    other = SlotEngine(EngineParams(slots=32, prime_bits=(60, 45, 45)))
    with pytest.raises(SerialError):
        load_ciphertext(other, tmp_path / "c.vrct")
    chain = SlotEngine(EngineParams(slots=64, prime_bits=(60, 40, 40)))
    with pytest.raises(SerialError):
        load_ciphertext(chain, tmp_path / "c.vrct")


def test_batch_round_trip(tmp_path, rng):
    eng = SlotEngine(EngineParams(slots=64, prime_bits=(60, 45)))
    lay = VirtualLayout(4, 16, 3, 4)
    imgs = rng.uniform(0, 1, size=(3, 3, 4))
    ct = pack_batch(eng, imgs, lay)
    write_batch(tmp_path / "b.vrct", ct, lay, 3, engine=eng)
    back, lay2, rows = load_batch(eng, tmp_path / "b.vrct")
    assert lay2 == lay and rows == 3
    np.testing.assert_array_equal(back.residues(), ct.residues())
    write_ciphertext(tmp_path / "plain.vrct", ct)
    with pytest.raises(SerialError):
        load_batch(eng, tmp_path / "plain.vrct")


def test_model_round_trip(tmp_path, rng):
    eng = SlotEngine(EngineParams(slots=32768, prime_bits=(60, 45)))
    kern = [Kernel(rng.uniform(-0.4, 0.4, (3, 3)), bias=0.05) for _ in range(4)]
    w = ModelWeights(kern, rng.uniform(-0.05, 0.05, (64, 2704)), rng.uniform(-0.1, 0.1, 64),
                     rng.uniform(-0.3, 0.3, (10, 64)), rng.uniform(-0.1, 0.1, 10), (0, 1, 0, 0), (0, 1, 0, 0))
    model = encode_model(eng, w)
    assert write_model(tmp_path / "m", model, engine=eng) == model.ciphertext_count == 52
    back = load_model(eng, tmp_path / "m")
    assert back.ciphertext_count == 52 and back.layout == model.layout
    assert (back.fc1_block, back.fc2_block, back.act1, back.act2) == (model.fc1_block, model.fc2_block, model.act1,
                                                                      model.act2)
    pairs = [(a, b) for sa, sb in zip(model.kernel_spans, back.kernel_spans)
             for a, b in zip(sa.span_cts + [sa.bias_ct], sb.span_cts + [sb.bias_ct])]
    pairs += [(a.ct, b.ct) for ra, rb in zip(model.fc1_tiles + model.fc2_tiles, back.fc1_tiles + back.fc2_tiles)
              for a, b in zip(ra, rb)]
    pairs += list(zip(model.fc1_bias_cts + model.fc2_bias_cts, back.fc1_bias_cts + back.fc2_bias_cts))
    assert len(pairs) == 52
    for a, b in pairs:
        np.testing.assert_array_equal(a.residues(), b.residues())
    with pytest.raises(SerialError):
        load_model(eng, tmp_path / "nothing-here")
