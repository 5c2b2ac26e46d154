"""Host-side breakdown of one end-to-end cfg-2 step (submit times of each public call, then wall)."""
import cProfile, pstats, sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer
from tools.workloads import cfg_matmul
a, b = cfg_matmul(2)
eng = CkksEngine(config_params(2))
def step(tt=None):
    t0 = time.perf_counter(); L = encode_left(eng, a, 64)
    t1 = time.perf_counter(); R = encode_right(eng, b, 64)
    t2 = time.perf_counter(); C = matmul_outer(eng, L, R)
    t3 = time.perf_counter(); out = C.decode(eng)
    t4 = time.perf_counter()
    if tt is not None: tt.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3))
    return out
for _ in range(10): step()
torch.cuda.synchronize()
tt = []
t0 = time.perf_counter()
for _ in range(50): step(tt)
wall = (time.perf_counter() - t0) / 50
m = np.median(np.array(tt), axis=0) * 1e3
print(f"wall {wall*1e3:.3f} ms/step; median submit ms: encL {m[0]:.3f} encR {m[1]:.3f} matmul {m[2]:.3f} decode(sync) {m[3]:.3f}")
pr = cProfile.Profile(); pr.enable()
for _ in range(50): step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
