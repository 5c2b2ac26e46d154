"""Host-side checks that need no GPU: the C-ABI library builds/loads and exports
every symbol include/vrhe.h declares, parameter/prime logic, meter semantics,
the modular-arithmetic header (compiled for the host), and the failure mode
without a GPU (no silent CPU fallback)."""

import ctypes
import json
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2512_18646_b200 import _lib
from paper_2512_18646_b200.engine import OpMeter, PlainMask
from paper_2512_18646_b200.errors import CapacityError, EngineError
from paper_2512_18646_b200.params import EngineParams, config_params, gen_primes, is_prime

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def libvrhe():
    if not _lib.LIB_PATH.exists():
        _lib.build()
    return ctypes.CDLL(str(_lib.LIB_PATH))


def test_abi_exports_every_header_symbol(libvrhe):
    header = (ROOT / "include" / "vrhe.h").read_text()
    declared = set(re.findall(r"\b(vr_[a-z0-9_]+)\s*\(", header))
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(libvrhe, name), f"{name} declared in vrhe.h but not exported"
    assert set(_lib.EXPORTED) == declared


def test_lib_loads_and_reports_errors(libvrhe):
    lib = _lib.load()
    h = ctypes.c_void_p()
    primes = (ctypes.c_uint64 * 2)(17, 97)
    rc = lib.vr_ctx_create(40, 1, primes, 0, 0, 0, ctypes.byref(h))  # bad log_n
    assert rc == 3
    assert b"log_n" in lib.vr_last_error()


def test_engine_refuses_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2512_18646_b200 import CkksEngine

    with pytest.raises(EngineError):
        CkksEngine(EngineParams(slots=4))


def test_params_reference_semantics(tmp_path):
    p = EngineParams(slots=8)
    assert p.log_n == 4 and p.n == 16
    with pytest.raises(EngineError):
        EngineParams(slots=3)
    with pytest.raises(EngineError):
        EngineParams(slots=1)
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"slots": 16, "logq": 200, "delta": 40, "bogus": 1}))
    with pytest.raises(EngineError):
        EngineParams.from_config(cfg)
    cfg.write_text(json.dumps({"slots": 16, "logq": 200, "delta": 40}))
    p = EngineParams.from_config(cfg)
    assert p.prime_bits == (60, 40, 40)


def test_primes_ntt_friendly():
    for cfg in (1, 2, 3, 4, 5):
        p = config_params(cfg)
        two_n = 2 * p.n
        assert len(set(p.primes)) == len(p.primes)
        for q, b in zip(p.primes, list(p.prime_bits) + [p.special_bits]):
            assert q % two_n == 1 and q.bit_length() == b and is_prime(q)
    # scale chain: s[l-1] = s[l]^2 / q[l]
    p = config_params(4)
    s = p.scale_chain()
    assert s[-1] == 2.0 ** 45
    for lv in range(p.levels, 0, -1):
        assert s[lv - 1] == (s[lv] * s[lv]) / float(p.primes[lv])


def test_meter_semantics():
    a = OpMeter(add_count=1, mul_count=2, max_depth=3)
    b = OpMeter(add_count=4, rot_count=1, max_depth=1)
    m = a.merged(b)
    assert (m.add_count, m.mul_count, m.rot_count, m.max_depth) == (5, 2, 1, 3)
    d = m.delta_since(a)
    assert (d.add_count, d.rot_count, d.max_depth) == (4, 1, 3)
    with pytest.raises(EngineError):
        PlainMask(np.array([0.5, 1.0]), role="filter")


HARNESS = r"""
#include <stdio.h>
#include <stdlib.h>
#include "modarith.cuh"
using namespace vr;
int main(int argc, char** argv) {
    unsigned long long q = strtoull(argv[1], 0, 10);
    unsigned __int128 r = (~(unsigned __int128)0) / q;
    Modulus m{q, (uint64_t)(r >> 64), (uint64_t)r};
    unsigned long long w = strtoull(argv[2], 0, 10);
    uint64_t wsh = (uint64_t)(((unsigned __int128)w << 64) / q);
    unsigned long long x, y, hi, lo;
    while (scanf("%llu %llu %llu %llu", &x, &y, &hi, &lo) == 4) {
        u128 z{lo, hi};
        printf("%llu %llu %llu %llu %llu\n", (unsigned long long)reduce128(z, m), (unsigned long long)mul_mod(x, y, m),
               (unsigned long long)mul_shoup(x, w, wsh, q), (unsigned long long)lift_centered(x, q, m),
               (unsigned long long)from_i64((int64_t)y, m));
    }
    return 0;
}
"""


def test_modarith_header_on_host(tmp_path):
    src = tmp_path / "h.cpp"
    src.write_text(HARNESS)
    exe = tmp_path / "h"
    subprocess.run(["g++", "-O2", "-std=c++17", f"-I{ROOT / 'paper_2512_18646_b200' / 'csrc'}", str(src), "-o", str(exe)],
                   check=True)
    rng = np.random.default_rng(3)
    for q in gen_primes(14, [60, 45, 40, 61]):
        w = int(rng.integers(0, q))
        rows = []
        for _ in range(400):
            x = int(rng.integers(0, q))
            y = int(rng.integers(-(2 ** 63), 2 ** 63 - 1))
            z = int(rng.integers(0, 2 ** 63)) * (2 ** 65) + int(rng.integers(0, 2 ** 63))
            z = min(z, 2 ** 128 - 1)
            rows.append((x, y % (2 ** 64), z >> 64, z & (2 ** 64 - 1), z, y))
        rows.append((q - 1, 2 ** 64 - 1, 2 ** 64 - 1, 2 ** 64 - 1, 2 ** 128 - 1, -1))
        rows.append((0, 2 ** 63, 0, 0, 0, -(2 ** 63)))  # INT64_MIN through from_i64
        rows.append((1, 2 ** 63 - 1, 0, 1, 1, 2 ** 63 - 1))
        inp = "\n".join(f"{x} {y} {hi} {lo}" for x, y, hi, lo, _, _ in rows)
        out = subprocess.run([str(exe), str(q), str(w)], input=inp, capture_output=True, text=True, check=True).stdout.split("\n")
        for (x, yu, hi, lo, z, ys), line in zip(rows, out):
            r128, mm, sh, lift, fi = (int(v) for v in line.split())
            assert r128 == z % q
            assert mm == (x * (yu % q)) % q
            assert sh == (x * w) % q
            assert lift == (x - q if x > q // 2 else x) % q
            assert fi == ys % q


def test_ct_batch_is_lazy_and_list_like():
    """CtBatch (the `cts` of encode_left / encode_right): Ciphertext objects and the pointer table come
    from base + i * stride, created on first access (no GPU needed for the bookkeeping)."""
    import torch

    from paper_2512_18646_b200.engine import CtBatch
    from paper_2512_18646_b200.multicipher import _OperandCache, _layout0, _storages

    out = torch.zeros((4, 2, 3, 8), dtype=torch.int64)
    b = CtBatch(out, 2, 2.0 ** 40, 0, ("grid", 2, 2), 7, 4, None)
    assert len(b) == 4 and b._items is None
    step = out.stride(0) * out.element_size()
    assert list(b.pointers()) == [out.data_ptr() + i * step for i in range(4)]
    assert b._items is None  # the pointer table did not create the ciphertexts
    assert [c._idx for c in b] == [0, 1, 2, 3] and b[1]._ptr == out.data_ptr() + step
    assert len(b + [1]) == 5 and len([0] + b) == 5 and _layout0(b) == ("grid", 2, 2)
    cache = _OperandCache(7, 2, 0, _storages(b), np_ptrs=b.pointers())
    assert list(cache.arr) == cache.ptrs == [c._ptr for c in b]
    # pending bookkeeping: a producer marks the batch, materialised items follow it
    owner = object()
    p = CtBatch(out, 2, 2.0 ** 40, 0, None, 7, 4, owner)
    assert all(c._pending is owner for c in p)
    p.set_pending(owner, None)
    assert p._pending is None and all(c._pending is None for c in p)


def test_failed_deferred_encryption_poisons_its_ciphertexts():
    """If the deferred launch raises, later uses of those ciphertexts raise as well (no garbage reads)."""
    import torch

    from paper_2512_18646_b200.engine import CtBatch, _FailedProducer
    from paper_2512_18646_b200.errors import EngineError

    out = torch.zeros((2, 2, 3, 8), dtype=torch.int64)
    owner = object()
    b = CtBatch(out, 2, 2.0 ** 40, 0, None, 7, 2, owner)
    cts = list(b)
    b.set_pending(owner, _FailedProducer("boom"))
    with pytest.raises(EngineError, match="boom"):
        cts[0].ptr()
    with pytest.raises(EngineError, match="boom"):
        b.order_on(object())
