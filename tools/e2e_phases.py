"""Device-time phases of the e2e cfg-2 step (events on the engine stream between public calls)."""
import sys; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer
from tools.workloads import cfg_matmul
a, b = cfg_matmul(2)
eng = CkksEngine(config_params(2))
s = torch.cuda.current_stream()
ph = {k: [] for k in ("h2d+encL", "encR", "matmul", "decode+d2h")}
for it in range(40):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    torch.cuda.synchronize()
    ev[0].record(s); L = encode_left(eng, a, 64)
    ev[1].record(s); R = encode_right(eng, b, 64)
    ev[2].record(s); C = matmul_outer(eng, L, R); eng.join()
    ev[3].record(s); out = C.decode(eng)
    ev[4].record(s); torch.cuda.synchronize()
    if it >= 10:
        for j, k in enumerate(ph):
            ph[k].append(ev[j].elapsed_time(ev[j + 1]) * 1e3)
print({k: round(float(np.median(v)), 1) for k, v in ph.items()}, "us; total", round(sum(float(np.median(v)) for v in ph.values()), 1))
import time
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    out = matmul_outer(eng, encode_left(eng, a, 64), encode_right(eng, b, 64)).decode(eng)
print("wall per e2e step", round((time.perf_counter() - t0) / 50 * 1e6, 1), "us")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(50):
    out = matmul_outer(eng, encode_left(eng, a, 64), encode_right(eng, b, 64)).decode(eng)
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(12)
