"""serial.py file format on the CPU (serial.py / test_serial.py:21-60 of the reference): bit-exact
round trip of residue payloads and the corrupt-file errors, with a host-side stand-in ciphertext."""

import numpy as np
import pytest

from paper_2512_18646_b200.serial import MAGIC, SerialError, read_ciphertext, write_ciphertext


class HostCt:
    def __init__(self, res, level, scale, depth=0, layout=None):
        self._res, self.level, self.scale, self.depth, self.layout = res, level, scale, depth, layout

    def residues(self):
        return self._res


def _ct(rng, n=16, level=2, degree=1):
    res = rng.integers(0, 2 ** 60, size=(degree + 1, level + 1, n), dtype=np.uint64)
    return HostCt(res, level, 2.0 ** 40 * 1.2345, depth=3, layout=("grid", 4, 4))


def test_round_trip_bit_exact(tmp_path, rng):
    ct = _ct(rng)
    p = tmp_path / "a.vrct"
    write_ciphertext(p, ct, meta={"k": 1})
    res, hdr = read_ciphertext(p)
    np.testing.assert_array_equal(res, ct.residues())
    assert float.fromhex(hdr["scale"]) == ct.scale
    assert (hdr["level"], hdr["degree"], hdr["depth"], hdr["slots"]) == (2, 1, 3, 8)
    assert tuple(hdr["layout"]) == ct.layout and hdr["meta"] == {"k": 1}
    ct2 = _ct(rng, degree=2, level=0)
    write_ciphertext(p, ct2)
    np.testing.assert_array_equal(read_ciphertext(p)[0], ct2.residues())


def test_rejects_garbage_and_truncation(tmp_path, rng):
    p = tmp_path / "g.vrct"
    p.write_bytes(b"not a ciphertext at all")
    with pytest.raises(SerialError):
        read_ciphertext(p)
    p.write_bytes(MAGIC + b"\x01")
    with pytest.raises(SerialError):
        read_ciphertext(p)
    write_ciphertext(p, _ct(rng))
    data = p.read_bytes()
    p.write_bytes(data[:-8])
    with pytest.raises(SerialError):
        read_ciphertext(p)
    p.write_bytes(MAGIC + (1000).to_bytes(4, "little") + b"{}")
    with pytest.raises(SerialError):
        read_ciphertext(p)
    p.write_bytes(MAGIC + (2).to_bytes(4, "little") + b"{}")
    with pytest.raises(SerialError):
        read_ciphertext(p)
