"""Host-side robustness of the GPU engine: stream semantics, context lifetime and
per-context launch configuration."""

import gc

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2512_18646_b200 import (CapacityError, CkksEngine, EngineError, EngineParams, config_params,  # noqa: E402
                                   encode_left, encode_right, matmul_outer)

TOL = 1e-3


def _small():
    return CkksEngine(EngineParams(slots=1024, prime_bits=(60, 40, 40), delta=40, seed=3))


def test_engine_runs_on_the_callers_current_stream():
    """Like a torch op, every call is ordered on torch.cuda.current_stream(): kernels, output
    allocations, the pinned H2D staging and the decode's D2H never straddle two streams."""
    eng = _small()
    x = np.random.default_rng(0).uniform(-1, 1, 1024)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        ct = eng.enc(x)
        sq = eng.mul(ct, ct)
        got = eng.dec(sq)
        assert eng._stream_ptr == side.cuda_stream
    np.testing.assert_allclose(got, x * x, atol=TOL)
    # back on the default stream, consuming ciphertexts made on the side stream
    torch.cuda.current_stream().wait_stream(side)
    got2 = eng.dec(eng.add(sq, ct))
    assert eng._stream_ptr == torch.cuda.current_stream().cuda_stream
    np.testing.assert_allclose(got2, x * x + x, atol=TOL)


def test_contexts_configure_their_own_kernels():
    """The dynamic shared-memory limits (tensor sum: 64 KB, cluster NTT) are raised per context:
    a second context created after the first is destroyed still launches them."""
    a, b = np.random.default_rng(1).uniform(-1, 1, (2, 64, 64))
    for _ in range(2):
        eng = CkksEngine(config_params(2))
        out = matmul_outer(eng, encode_left(eng, a, 64), encode_right(eng, b, 64))
        assert float(np.max(np.abs(out.decode(eng) - a @ b))) < TOL
        del eng, out
        gc.collect()


def test_bad_parameters_raise_engine_error():
    from paper_2512_18646_b200 import _lib

    lib = _lib.load()
    import ctypes

    h = ctypes.c_void_p()
    primes = (ctypes.c_uint64 * 3)(7, 11, 13)  # not 1 mod 2N
    with pytest.raises(EngineError):
        _lib.check(lib.vr_ctx_create(10, 2, primes, 0, 1, 0, ctypes.byref(h)))
    assert not h.value


def test_cmul_constant_overflow_is_a_capacity_error():
    eng = _small()
    ct = eng.enc([1.0, 2.0])
    with pytest.raises(CapacityError):
        eng.cmul(eng.mask(np.full(eng.slots, 2.0 ** 30)), ct)  # 2^30 * 2^40 does not fit int64


@pytest.mark.parametrize("cfg", [1, 2])
def test_matmul_outer_graph_replay_bit_exact(cfg):
    """Repeated products of the same operands: the first call per (slot, operands) runs eagerly, the
    second records the slot's CUDA graph, later ones replay it asynchronously on the slot streams
    (three in flight).  Every result is identical to the first, whatever happens to the outputs."""
    eng = CkksEngine(config_params(cfg))
    dim = 8 if cfg == 1 else 64
    a, b = np.random.default_rng(cfg).uniform(-1, 1, (2, dim, dim))
    left, right = encode_left(eng, a, dim), encode_right(eng, b, dim)
    first = matmul_outer(eng, left, right)
    want = first.ct.residues()
    np.testing.assert_allclose(first.decode(eng), a @ b, atol=TOL)
    kept = []
    for i in range(24):
        out = matmul_outer(eng, left, right)
        if i % 3 == 0:
            kept.append(out)  # held while later products are in flight
        elif i % 3 == 1:
            del out  # dropped before it completes: the allocator must not hand the buffer out early
        else:
            junk = torch.full((2, eng.L, eng.N), 7, dtype=torch.int64, device=eng.device)  # reuse pressure
            np.testing.assert_array_equal(out.ct.residues(), want)
            del junk
    for out in kept:
        np.testing.assert_array_equal(out.ct.residues(), want)
    eng.join()


def test_async_results_feed_later_ops():
    """An asynchronous product used directly by the next engine call (decode, add) is complete first."""
    eng = CkksEngine(config_params(2))
    a, b = np.random.default_rng(5).uniform(-1, 1, (2, 64, 64))
    left, right = encode_left(eng, a, 64), encode_right(eng, b, 64)
    outs = [matmul_outer(eng, left, right) for _ in range(8)]
    total = outs[0].ct
    for o in outs[1:]:
        total = eng.add(total, o.ct)
    got = eng.dec(total)[: 64 * 64].reshape(64, 64)
    np.testing.assert_allclose(got, 8 * (a @ b), atol=8 * TOL)


def test_decode_async_pipeline_matches_decode():
    """Several encrypt -> matmul_outer -> decode_async steps in flight (fresh operands every step, so
    the slot graphs are re-pointed at new operands each time): every result equals A B."""
    eng = CkksEngine(config_params(2))
    rng = np.random.default_rng(9)
    mats = [rng.uniform(-1, 1, (2, 64, 64)) for _ in range(20)]
    futs = [matmul_outer(eng, encode_left(eng, a, 64), encode_right(eng, b, 64)).decode_async(eng) for a, b in mats]
    for (a, b), f in zip(mats, futs):
        np.testing.assert_allclose(f.result(), a @ b, atol=TOL)
