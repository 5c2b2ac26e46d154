"""Host cost of one config-2 matmul_outer call (async path): whole Python call, raw C-ABI call,
and a cProfile of the Python layer.  python tools/host_probe.py"""
import cProfile, ctypes, pstats, sys, time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2512_18646_b200 import CkksEngine, _lib, config_params, encode_left, encode_right, matmul_outer
from paper_2512_18646_b200.multicipher import _fast_operand

eng = CkksEngine(config_params(2))
a, b = np.random.default_rng(1).uniform(-1, 1, (2, 64, 64))
L, R = encode_left(eng, a, 64), encode_right(eng, b, 64)
for _ in range(30):
    out = matmul_outer(eng, L, R)
eng.join(); torch.cuda.synchronize()


def burst(fn, k=8):
    t = 0.0
    for _ in range(10):
        t0 = time.perf_counter()
        for _ in range(k):
            fn()
        t += time.perf_counter() - t0
        eng.join(); torch.cuda.synchronize()
    return t / (10 * k) * 1e6


print(f"matmul_outer (python + C): {burst(lambda: matmul_outer(eng, L, R)):.1f} us/call")
fl, fr = _fast_operand(eng, L), _fast_operand(eng, R)
outs = torch.empty((1, 2, eng.L, eng.N), dtype=torch.int64, device="cuda")
op = _lib.row_ptrs(outs, 1)
slot = ctypes.c_void_p()
h = eng.handle
print(f"vr_matmul_outer_async alone: {burst(lambda: eng._lib.vr_matmul_outer_async(h, fl.arr, fr.arr, 64, 1, eng.L, op, ctypes.byref(slot))):.1f} us/call")
print(f"torch.empty: {burst(lambda: torch.empty((1, 2, eng.L, eng.N), dtype=torch.int64, device='cuda')):.1f} us/call")
print(f"engine.handle: {burst(lambda: eng.handle):.1f} us/call")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    out = matmul_outer(eng, L, R)
    if _ % 8 == 7:
        eng.join(); torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
