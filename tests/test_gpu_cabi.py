"""The C-ABI on its own (include/vrhe.h), driven through ctypes with no PyTorch tensors: what a
cgo / JNI / plain-ctypes binding of the packedhe engine would do.

* vr_ct objects: host doubles -> vr_encrypt_host -> vr_matmul_outer_ct -> vr_decrypt_host; decoded
  A B within 1e-3 (multicipher.py:62-103) and residues bit-identical to the CPU oracle's matmul
  on the same inputs; upload/download round trips; layout errors map to status 2.
* the native NCCL communicator at world size 1 (vr_comm_*, vr_sum_partials): the sharded config-5a
  path through it equals the unsharded product bit for bit.
"""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.engine import OCt, OracleEngine  # noqa: E402
from paper_2512_18646_b200 import LayoutError, _lib, config_params  # noqa: E402

TOL = 1e-3


class RawEngine:
    """Minimal ctypes-only client of libvrhe.so."""

    def __init__(self, params):
        self.lib = _lib.load()
        self.p = params
        primes = (ctypes.c_uint64 * len(params.primes))(*params.primes)
        self.h = ctypes.c_void_p()
        _lib.check(self.lib.vr_ctx_create(params.log_n, len(params.prime_bits), primes, params.seed, 1, 0, ctypes.byref(self.h)))
        self.L, self.N, self.S = params.levels, params.n, params.slots

    def alloc(self, level, scale=1.0):
        ct = ctypes.c_void_p()
        _lib.check(self.lib.vr_ct_alloc(self.h, level, 1, scale, ctypes.byref(ct)))
        return ct

    def encrypt(self, rows, nonce0):
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        cts = [self.alloc(self.L) for _ in range(rows.shape[0])]
        arr = (ctypes.c_void_p * len(cts))(*[c.value for c in cts])
        _lib.check(self.lib.vr_encrypt_host(self.h, rows.ctypes.data, rows.shape[0], rows.shape[1], self.p.scale, nonce0, arr))
        return cts

    def decrypt(self, cts):
        out = np.empty((len(cts), self.S))
        arr = (ctypes.c_void_p * len(cts))(*[c.value for c in cts])
        _lib.check(self.lib.vr_decrypt_host(self.h, arr, len(cts), out.ctypes.data))
        return out

    def residues(self, ct):
        lvl = self.lib.vr_ct_level(ct)
        host = np.empty((2, lvl + 1, self.N), dtype=np.uint64)
        _lib.check(self.lib.vr_ct_download(self.h, ct, host.ctypes.data))
        return host

    def close(self, cts):
        for c in cts:
            _lib.check(self.lib.vr_ct_free(self.h, c))
        _lib.check(self.lib.vr_ctx_destroy(self.h))


def test_c_abi_matmul_round_trip_bit_exact():
    p = config_params(1)
    eng, orc = RawEngine(p), OracleEngine.from_params(p)
    rng = np.random.default_rng(0)
    a, b = rng.uniform(-1, 1, (2, 8, 8))
    Lrows = np.stack([np.repeat(a[:, k], 8) for k in range(8)])  # encode_left layout
    Rrows = np.stack([np.tile(b[k, :], 8) for k in range(8)])  # encode_right layout
    L = eng.encrypt(Lrows, 0)
    R = eng.encrypt(Rrows, 8)
    out = eng.alloc(eng.L - 1)
    _lib.check(eng.lib.vr_matmul_outer_ct(eng.h, (ctypes.c_void_p * 8)(*[c.value for c in L]),
                                          (ctypes.c_void_p * 8)(*[c.value for c in R]), 8, 1,
                                          (ctypes.c_void_p * 1)(out.value)))
    got = eng.decrypt([out])[0][:64].reshape(8, 8)
    np.testing.assert_allclose(got, a @ b, atol=TOL)
    assert abs(eng.lib.vr_ct_scale(out) - p.scale_chain()[eng.L - 1]) < 1e-6 * p.scale_chain()[eng.L - 1]
    oL = [orc.enc(r) for r in Lrows]
    oR = [orc.enc(r) for r in Rrows]
    for c, o in zip(L[:2] + R[:2], oL[:2] + oR[:2]):
        np.testing.assert_array_equal(eng.residues(c), o.data)
    want = orc.matmul_outer_blocks([oL], oR)[0]
    np.testing.assert_array_equal(eng.residues(out), want.data)
    # upload / download round trip
    blob = eng.residues(L[3])
    tmp = eng.alloc(eng.L)
    _lib.check(eng.lib.vr_ct_upload(eng.h, tmp, blob.ctypes.data))
    np.testing.assert_array_equal(eng.residues(tmp), blob)
    # wrong output level -> LayoutError (status 2)
    bad = eng.alloc(eng.L)
    with pytest.raises(LayoutError):
        _lib.check(eng.lib.vr_matmul_outer_ct(eng.h, (ctypes.c_void_p * 8)(*[c.value for c in L]),
                                              (ctypes.c_void_p * 8)(*[c.value for c in R]), 8, 1,
                                              (ctypes.c_void_p * 1)(bad.value)))
    eng.close(L + R + [out, tmp, bad])


def test_native_comm_world1_sharded_equals_unsharded():
    from paper_2512_18646_b200 import CkksEngine, encode_left, encode_right, matmul_outer_blocks
    from paper_2512_18646_b200.dist import NativeComm, encode_operands_sharded, matmul_outer_sharded_owned

    p = config_params(2)
    eng = CkksEngine(p)
    rng = np.random.default_rng(4)
    a, b = rng.uniform(-1, 1, (2, 64, 64))
    blocks = [a[32 * i: 32 * (i + 1)] for i in range(2)]
    ref = [c.residues() for c in matmul_outer_blocks(eng, [encode_left(eng, blk, 64) for blk in blocks],
                                                     encode_right(eng, b, 32))]
    comm = NativeComm(eng, NativeComm.unique_id(eng), 0, 1)
    ls, rs = encode_operands_sharded(eng, blocks, b, 0, 64)
    outs = matmul_outer_sharded_owned(eng, ls, rs, comm=comm)
    assert sorted(outs) == [0, 1]
    for bi, r in enumerate(ref):
        np.testing.assert_array_equal(outs[bi].residues(), r)
    comm.close()
