"""ctypes bindings for the CPU RNS-CKKS residue oracle (oracle/ckks_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg.  The product package never
imports this module.

``OracleCkks`` exposes the raw residue operations on numpy uint64 arrays with
the same layouts as the CUDA library ([deg+1][level+1][N], NTT domain).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libckks_oracle.so"
_lib = None

u64p = ctypes.POINTER(ctypes.c_uint64)
i64p = ctypes.POINTER(ctypes.c_int64)
dblp = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> Path:
    src = _HERE / "ckks_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB_PATH))
        vp = ctypes.c_void_p
        L.orc_gen_primes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int), u64p]
        L.orc_create.restype = vp
        L.orc_create.argtypes = [ctypes.c_int, ctypes.c_int, u64p, ctypes.c_uint64, ctypes.c_int]
        L.orc_destroy.argtypes = [vp]
        L.orc_stream_key.restype = ctypes.c_uint64
        L.orc_stream_key.argtypes = [ctypes.c_uint64] * 4
        L.orc_build_cdt.argtypes = [u64p]
        L.orc_get_tables.argtypes = [vp, ctypes.c_int, u64p, u64p]
        L.orc_get_secret.argtypes = [vp, ctypes.POINTER(ctypes.c_int8)]
        L.orc_get_pk.argtypes = [vp, u64p]
        L.orc_get_relin_key.argtypes = [vp, u64p]
        L.orc_get_galois_key.argtypes = [vp, ctypes.c_uint32, u64p]
        L.orc_encode_coeffs.argtypes = [vp, dblp, ctypes.c_int, ctypes.c_double, i64p]
        L.orc_decode_coeffs.argtypes = [vp, i64p, ctypes.c_double, dblp, dblp]
        L.orc_encode.argtypes = [vp, dblp, ctypes.c_int, ctypes.c_int, ctypes.c_double, u64p]
        L.orc_encrypt.argtypes = [vp, dblp, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_uint64, u64p]
        L.orc_decrypt_coeffs.argtypes = [vp, u64p, ctypes.c_int, ctypes.c_int, i64p]
        L.orc_decrypt_decode.argtypes = [vp, u64p, ctypes.c_int, ctypes.c_int, ctypes.c_double, dblp]
        for name in ("orc_add", "orc_sub"):
            getattr(L, name).argtypes = [vp, u64p, u64p, ctypes.c_int, ctypes.c_int, u64p]
        L.orc_tensor.argtypes = [vp, u64p, u64p, ctypes.c_int, u64p]
        L.orc_mul_plain.argtypes = [vp, u64p, u64p, ctypes.c_int, ctypes.c_int, u64p]
        L.orc_mul_scalar.argtypes = [vp, u64p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, u64p]
        L.orc_add_const.argtypes = [vp, u64p, ctypes.c_int64, ctypes.c_int]
        L.orc_drop_level.argtypes = [vp, u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, u64p]
        L.orc_rescale.argtypes = [vp, u64p, ctypes.c_int, ctypes.c_int, u64p]
        L.orc_keyswitch.argtypes = [vp, u64p, ctypes.c_int, u64p, u64p]
        L.orc_relin.argtypes = [vp, u64p, ctypes.c_int, u64p]
        L.orc_relin_rescale.argtypes = [vp, u64p, ctypes.c_int, u64p]
        L.orc_galois_elt.restype = ctypes.c_uint32
        L.orc_galois_elt.argtypes = [vp, ctypes.c_int64]
        L.orc_rotate.argtypes = [vp, u64p, ctypes.c_int, ctypes.c_int64, u64p]
        L.orc_mul.argtypes = [vp, u64p, u64p, ctypes.c_int, u64p]
        L.orc_matmul_outer.argtypes = [vp, ctypes.POINTER(u64p), ctypes.POINTER(u64p), ctypes.c_int, ctypes.c_int, u64p]
        L.orc_conv_columns.argtypes = [
            vp, ctypes.POINTER(u64p), ctypes.c_int, ctypes.c_int, ctypes.c_int, i64p, u64p, ctypes.c_int,
            ctypes.POINTER(ctypes.c_int), ctypes.c_int, u64p, ctypes.c_int, ctypes.POINTER(u64p),
        ]
        L.orc_poly_activation.argtypes = [vp, u64p, ctypes.c_int, i64p, ctypes.c_int, u64p]
        L.orc_ntt_limb.argtypes = [vp, ctypes.c_int, u64p]
        L.orc_intt_limb.argtypes = [vp, ctypes.c_int, u64p]
        L.orc_galois_perm.argtypes = [vp, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32)]
        _lib = L
    return _lib


def _p(a: np.ndarray, ptype=u64p):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ptype)


def gen_primes(log_n: int, bits) -> np.ndarray:
    bits = list(bits)
    out = np.zeros(len(bits), dtype=np.uint64)
    arr = (ctypes.c_int * len(bits))(*bits)
    rc = lib().orc_gen_primes(log_n, len(bits), arr, _p(out))
    if rc != 0:
        raise ValueError(f"prime generation failed ({rc})")
    return out


def build_cdt() -> np.ndarray:
    out = np.zeros(32, dtype=np.uint64)
    lib().orc_build_cdt(_p(out))
    return out


def stream_key(seed, dom, a, b) -> int:
    return int(lib().orc_stream_key(seed, dom, a, b))


class OracleCkks:
    """Residue-level CPU CKKS context (same primes, seed and layouts as the GPU)."""

    def __init__(self, log_n: int, primes, seed: int, sym_enc: bool = False):
        self.log_n = log_n
        self.n = 1 << log_n
        self.slots = self.n // 2
        self.primes = np.ascontiguousarray(np.asarray(primes, dtype=np.uint64))
        self.L = len(self.primes) - 2
        self.seed = seed
        self._c = lib().orc_create(log_n, self.L + 1, _p(self.primes), seed, int(sym_enc))
        if not self._c:
            raise ValueError("oracle context creation failed")

    def __del__(self):
        if getattr(self, "_c", None):
            lib().orc_destroy(self._c)
            self._c = None

    # -- shapes --------------------------------------------------------
    def _ct(self, deg: int, level: int) -> np.ndarray:
        return np.zeros((deg + 1, level + 1, self.n), dtype=np.uint64)

    @staticmethod
    def level_of(ct: np.ndarray) -> int:
        return ct.shape[1] - 1

    # -- tables / keys --------------------------------------------------
    def tables(self, pidx: int):
        a = np.zeros(self.n, dtype=np.uint64)
        b = np.zeros(self.n, dtype=np.uint64)
        lib().orc_get_tables(self._c, pidx, _p(a), _p(b))
        return a, b

    def secret(self) -> np.ndarray:
        s = np.zeros(self.n, dtype=np.int8)
        lib().orc_get_secret(self._c, s.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)))
        return s

    def public_key(self) -> np.ndarray:
        out = np.zeros((2, self.L + 1, self.n), dtype=np.uint64)
        lib().orc_get_pk(self._c, _p(out))
        return out

    def relin_key(self) -> np.ndarray:
        out = np.zeros((self.L + 1, 2, self.L + 2, self.n), dtype=np.uint64)
        lib().orc_get_relin_key(self._c, _p(out))
        return out

    def galois_key(self, g: int) -> np.ndarray:
        out = np.zeros((self.L + 1, 2, self.L + 2, self.n), dtype=np.uint64)
        lib().orc_get_galois_key(self._c, g, _p(out))
        return out

    def galois_elt(self, steps: int) -> int:
        return int(lib().orc_galois_elt(self._c, steps))

    def galois_perm(self, g: int) -> np.ndarray:
        out = np.zeros(self.n, dtype=np.uint32)
        lib().orc_galois_perm(self._c, g, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
        return out

    # -- NTT -------------------------------------------------------------
    def ntt(self, a: np.ndarray, pidx: int) -> np.ndarray:
        out = np.ascontiguousarray(a, dtype=np.uint64).copy()
        lib().orc_ntt_limb(self._c, pidx, _p(out))
        return out

    def intt(self, a: np.ndarray, pidx: int) -> np.ndarray:
        out = np.ascontiguousarray(a, dtype=np.uint64).copy()
        lib().orc_intt_limb(self._c, pidx, _p(out))
        return out

    # -- encode / encrypt / decrypt ------------------------------------
    def encode_coeffs(self, values, scale: float) -> np.ndarray:
        v = np.ascontiguousarray(np.asarray(values, dtype=np.float64).reshape(-1))
        out = np.zeros(self.n, dtype=np.int64)
        lib().orc_encode_coeffs(self._c, _p(v, dblp), v.size, scale, _p(out, i64p))
        return out

    def decode_coeffs(self, m: np.ndarray, scale: float) -> np.ndarray:
        m = np.ascontiguousarray(m, dtype=np.int64)
        re = np.zeros(self.slots)
        im = np.zeros(self.slots)
        lib().orc_decode_coeffs(self._c, _p(m, i64p), scale, _p(re, dblp), _p(im, dblp))
        return re + 1j * im

    def encode(self, values, level: int, scale: float) -> np.ndarray:
        v = np.ascontiguousarray(np.asarray(values, dtype=np.float64).reshape(-1))
        out = np.zeros((level + 1, self.n), dtype=np.uint64)
        lib().orc_encode(self._c, _p(v, dblp), v.size, level, scale, _p(out))
        return out

    def encrypt(self, values, level: int, scale: float, nonce: int) -> np.ndarray:
        v = np.ascontiguousarray(np.asarray(values, dtype=np.float64).reshape(-1))
        out = self._ct(1, level)
        lib().orc_encrypt(self._c, _p(v, dblp), v.size, level, scale, nonce, _p(out))
        return out

    def decrypt_coeffs(self, ct: np.ndarray) -> np.ndarray:
        ct = np.ascontiguousarray(ct)
        out = np.zeros(self.n, dtype=np.int64)
        lib().orc_decrypt_coeffs(self._c, _p(ct), ct.shape[0] - 1, ct.shape[1] - 1, _p(out, i64p))
        return out

    def decrypt_decode(self, ct: np.ndarray, scale: float) -> np.ndarray:
        ct = np.ascontiguousarray(ct)
        out = np.zeros(self.slots)
        lib().orc_decrypt_decode(self._c, _p(ct), ct.shape[0] - 1, ct.shape[1] - 1, scale, _p(out, dblp))
        return out

    # -- ring ops --------------------------------------------------------
    def add(self, a, b):
        out = np.zeros_like(a)
        lib().orc_add(self._c, _p(a), _p(b), a.shape[0] - 1, a.shape[1] - 1, _p(out))
        return out

    def sub(self, a, b):
        out = np.zeros_like(a)
        lib().orc_sub(self._c, _p(a), _p(b), a.shape[0] - 1, a.shape[1] - 1, _p(out))
        return out

    def tensor(self, a, b):
        lvl = a.shape[1] - 1
        out = self._ct(2, lvl)
        lib().orc_tensor(self._c, _p(a), _p(b), lvl, _p(out))
        return out

    def mul_plain(self, ct, pt):
        out = np.zeros_like(ct)
        lib().orc_mul_plain(self._c, _p(ct), _p(np.ascontiguousarray(pt)), ct.shape[0] - 1, ct.shape[1] - 1, _p(out))
        return out

    def mul_scalar(self, ct, s: int):
        out = np.zeros_like(ct)
        lib().orc_mul_scalar(self._c, _p(ct), int(s), ct.shape[0] - 1, ct.shape[1] - 1, _p(out))
        return out

    def add_const(self, ct, s: int):
        out = ct.copy()
        lib().orc_add_const(self._c, _p(out), int(s), ct.shape[1] - 1)
        return out

    def drop_level(self, ct, to: int):
        out = self._ct(ct.shape[0] - 1, to)
        lib().orc_drop_level(self._c, _p(ct), ct.shape[0] - 1, ct.shape[1] - 1, to, _p(out))
        return out

    def rescale(self, ct):
        lvl = ct.shape[1] - 1
        out = self._ct(ct.shape[0] - 1, lvl - 1)
        lib().orc_rescale(self._c, _p(ct), ct.shape[0] - 1, lvl, _p(out))
        return out

    def keyswitch(self, poly, key):
        lvl = poly.shape[0] - 1
        out = self._ct(1, lvl)
        lib().orc_keyswitch(self._c, _p(np.ascontiguousarray(poly)), lvl, _p(key), _p(out))
        return out

    def relin(self, d3):
        lvl = d3.shape[1] - 1
        out = self._ct(1, lvl)
        lib().orc_relin(self._c, _p(d3), lvl, _p(out))
        return out

    def relin_rescale(self, d3):
        lvl = d3.shape[1] - 1
        out = self._ct(1, lvl - 1)
        lib().orc_relin_rescale(self._c, _p(np.ascontiguousarray(d3)), lvl, _p(out))
        return out

    def rotate(self, ct, steps: int):
        out = np.zeros_like(ct)
        lib().orc_rotate(self._c, _p(ct), ct.shape[1] - 1, int(steps), _p(out))
        return out

    def mul(self, a, b):
        lvl = a.shape[1] - 1
        out = self._ct(1, lvl - 1)
        lib().orc_mul(self._c, _p(a), _p(b), lvl, _p(out))
        return out

    # -- fused drivers -----------------------------------------------------
    def matmul_outer(self, Ls, Rs):
        lvl = Ls[0].shape[1] - 1
        n = len(Ls)
        la = (u64p * n)(*[_p(x) for x in Ls])
        ra = (u64p * n)(*[_p(x) for x in Rs])
        out = self._ct(1, lvl - 1)
        lib().orc_matmul_outer(self._c, la, ra, n, lvl, _p(out))
        return out

    def conv_columns(self, X, C, W, k, w_int, bias_res, F, out_cols, mask_pt):
        """X: list of C*W cts; w_int: int64 [F][C][k][k]; bias_res: uint64 [F][l+1] residues."""
        lvl = X[0].shape[1] - 1
        xa = (u64p * len(X))(*[_p(x) for x in X])
        w_int = np.ascontiguousarray(w_int, dtype=np.int64)
        bias_res = np.ascontiguousarray(bias_res, dtype=np.uint64)
        cols = (ctypes.c_int * len(out_cols))(*[int(c) for c in out_cols])
        Y = [self._ct(1, lvl - 1) for _ in range(F * len(out_cols))]
        ya = (u64p * len(Y))(*[_p(y) for y in Y])
        lib().orc_conv_columns(
            self._c, xa, C, W, k, _p(w_int, i64p), _p(bias_res), F, cols, len(out_cols),
            _p(np.ascontiguousarray(mask_pt)), lvl, ya,
        )
        return Y

    def poly_activation(self, x, kc, c3_zero: bool):
        lvl = x.shape[1] - 1
        kc = np.ascontiguousarray(np.asarray(kc, dtype=np.int64))
        out = self._ct(1, lvl - 2)
        lib().orc_poly_activation(self._c, _p(x), lvl, _p(kc, i64p), int(c3_zero), _p(out))
        return out
