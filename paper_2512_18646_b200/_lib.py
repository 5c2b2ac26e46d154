"""ctypes binding of libvrhe.so (the C-ABI in include/vrhe.h).

There is no fallback: if the CUDA library is missing or no GPU is visible the
engine raises immediately.  Status codes map to the reference's exception
classes (engine.py:32-41).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

from .errors import CapacityError, EngineError, LayoutError

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libvrhe.so"
_lib = None

c_u64p = ctypes.POINTER(ctypes.c_uint64)
c_vp = ctypes.c_void_p
c_vpp = ctypes.POINTER(ctypes.c_void_p)

# name -> argtypes (restype int unless noted)
_SIGS = {
    "vr_ctx_create": [ctypes.c_int, ctypes.c_int, c_u64p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(c_vp)],
    "vr_ctx_destroy": [c_vp],
    "vr_set_stream": [c_vp, c_vp],
    "vr_fork_stream": [c_vp, c_vp],
    "vr_sync": [c_vp],
    "vr_gen_relin_key": [c_vp],
    "vr_galois_elt": [c_vp, ctypes.c_int64, ctypes.POINTER(ctypes.c_uint32)],
    "vr_gen_galois_key": [c_vp, ctypes.c_uint32],
    "vr_export_secret": [c_vp, c_u64p],
    "vr_export_public_key": [c_vp, c_u64p],
    "vr_export_relin_key": [c_vp, c_u64p],
    "vr_export_galois_key": [c_vp, ctypes.c_uint32, c_u64p],
    "vr_ntt": [c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int],
    "vr_encode": [c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, c_vp],
    "vr_encode_coeffs": [c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_double, c_vp],
    "vr_encrypt": [c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_uint64, c_vp],
    "vr_encrypt_strided": [c_vp, c_vp, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_int, ctypes.c_int,
                           ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_uint64, c_vp],
    "vr_encrypt_strided2": [c_vp, c_vp, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_int, ctypes.c_int,
                            ctypes.c_int, c_vp, c_vp, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_int,
                            ctypes.c_int, ctypes.c_int, c_vp, ctypes.c_int, ctypes.c_double, ctypes.c_uint64],
    "vr_encrypt_strided_host": [c_vp, c_vp, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong,
                                ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                ctypes.c_uint64, c_vp],
    "vr_encrypt_strided2_host": [c_vp, c_vp, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong,
                                 ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_vp, c_vp, ctypes.c_longlong,
                                 ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_int,
                                 ctypes.c_int, ctypes.c_int, c_vp, ctypes.c_int, ctypes.c_double, ctypes.c_uint64],
    "vr_decode_submit": [c_vp, c_vpp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                         ctypes.POINTER(ctypes.c_double), ctypes.c_int, c_vp, ctypes.POINTER(ctypes.c_int)],
    "vr_decode_wait": [c_vp, ctypes.c_int, c_vp],
    "vr_decrypt_decode": [c_vp, c_vpp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                          ctypes.POINTER(ctypes.c_double), ctypes.c_int, c_vp, c_vp],
    "vr_add": [c_vp, c_vpp, c_vpp, c_vpp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int],
    "vr_tensor": [c_vp, c_vpp, c_vpp, c_vpp, ctypes.c_int, ctypes.c_int],
    "vr_relin": [c_vp, c_vpp, c_vpp, ctypes.c_int, ctypes.c_int],
    "vr_rescale": [c_vp, c_vpp, c_vpp, ctypes.c_int, ctypes.c_int, ctypes.c_int],
    "vr_relin_rescale": [c_vp, c_vpp, c_vpp, ctypes.c_int, ctypes.c_int],
    "vr_mul": [c_vp, c_vpp, c_vpp, c_vpp, ctypes.c_int, ctypes.c_int],
    "vr_mul_plain": [c_vp, c_vpp, c_vpp, c_vpp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int],
    "vr_mul_scalar": [c_vp, c_vpp, ctypes.c_int64, c_vpp, ctypes.c_int, ctypes.c_int, ctypes.c_int],
    "vr_add_const": [c_vp, c_vpp, ctypes.c_int64, ctypes.c_int, ctypes.c_int],
    "vr_drop_level": [c_vp, c_vpp, c_vpp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int],
    "vr_rotate": [c_vp, c_vpp, c_vpp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)],
    "vr_keyswitch": [c_vp, c_vp, ctypes.c_int, ctypes.c_uint32, c_vp],
    "vr_mod_reduce": [c_vp, c_vp, ctypes.c_longlong, ctypes.c_int],
    "vr_bench_butterflies": [c_vp, ctypes.c_int, ctypes.c_int, c_vp],
    "vr_bench_butterflies_f64": [c_vp, ctypes.c_int, ctypes.c_int, c_vp],
    "vr_matmul_outer": [c_vp, c_vpp, c_vpp, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_vpp],
    "vr_matmul_outer_many": [c_vp, c_vpp, c_vpp, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_vpp],
    "vr_tensor_sum": [c_vp, c_vpp, c_vpp, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_vpp],
    "vr_matmul_outer_async": [c_vp, c_vpp, c_vpp, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_vpp, ctypes.POINTER(c_vp)],
    "vr_join": [c_vp],
    "vr_async_slot": [c_vp, ctypes.POINTER(c_vp)],
    "vr_ct_alloc": [c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.POINTER(c_vp)],
    "vr_ct_free": [c_vp, c_vp],
    "vr_ct_upload": [c_vp, c_vp, c_vp],
    "vr_ct_download": [c_vp, c_vp, c_vp],
    "vr_encrypt_host": [c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_uint64, c_vpp],
    "vr_decrypt_host": [c_vp, c_vpp, ctypes.c_int, c_vp],
    "vr_matmul_outer_ct": [c_vp, c_vpp, c_vpp, ctypes.c_int, ctypes.c_int, c_vpp],
    "vr_comm_unique_id": [c_vp],
    "vr_comm_init": [c_vp, c_vp, ctypes.c_int, ctypes.c_int],
    "vr_comm_destroy": [c_vp],
    "vr_sum_partials": [c_vp, c_vp, ctypes.c_longlong, ctypes.c_int, ctypes.c_int],
    "vr_tensor_sum_mode": [c_vp, c_vpp, c_vpp, ctypes.c_int, ctypes.c_int, c_vp, ctypes.c_int],
    "vr_conv_columns": [c_vp, c_vpp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                        c_u64p, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int, c_vp,
                        ctypes.c_int, c_vpp],
    "vr_pt_matvec": [c_vp, c_vpp, ctypes.c_int, c_vpp, ctypes.c_int, ctypes.c_int, c_vpp],
    "vr_poly_activation": [c_vp, c_vpp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_int, c_vpp],
}

_ACCESSORS = {"vr_ct_data": (c_vp, [c_vp]), "vr_ct_level": (ctypes.c_int, [c_vp]), "vr_ct_degree": (ctypes.c_int, [c_vp]),
              "vr_ct_scale": (ctypes.c_double, [c_vp])}

EXPORTED = tuple(_SIGS) + tuple(_ACCESSORS) + ("vr_last_error", "vr_launch_count")


def build(force: bool = False) -> Path:
    """Compile libvrhe.so in-tree with nvcc for sm_100a (make -C csrc)."""
    csrc = _PKG / "csrc"
    args = ["make", "-s", "-C", str(csrc), f"-j{os.cpu_count() or 4}"]
    if force:
        subprocess.run(["make", "-s", "-C", str(csrc), "clean"], check=True)
    subprocess.run(args, check=True)
    return LIB_PATH


def load():
    """Load libvrhe.so; raises EngineError if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise EngineError(
            f"CUDA extension {LIB_PATH} is missing; build it with __graft_entry__.build() "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, argtypes in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = ctypes.c_int
    for name, (res, argtypes) in _ACCESSORS.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = res
    lib.vr_last_error.restype = ctypes.c_char_p
    lib.vr_last_error.argtypes = []
    lib.vr_launch_count.restype = ctypes.c_ulonglong
    lib.vr_launch_count.argtypes = []
    _lib = lib
    return lib


_ERRORS = {1: CapacityError, 2: LayoutError, 3: EngineError}


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = _lib.vr_last_error().decode(errors="replace") if _lib is not None else "libvrhe not loaded"
    exc = _ERRORS.get(rc)
    if exc is None:
        raise RuntimeError(f"libvrhe CUDA error: {msg}")
    raise exc(msg)


def ptr_array(ptrs):
    """Host array of device pointers for a pointer-table argument."""
    ptrs = list(ptrs)
    return (ctypes.c_void_p * max(1, len(ptrs)))(*ptrs)


def row_ptrs(t, count=None):
    """ptr_array of the leading-index rows of a contiguous device tensor (no per-row views)."""
    base, step = t.data_ptr(), t.stride(0) * t.element_size()
    n = t.shape[0] if count is None else count
    return (ctypes.c_void_p * max(1, n))(*[base + i * step for i in range(n)])
