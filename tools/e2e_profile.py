"""Launch list of one end-to-end cfg-2 step (host A,B -> encrypt -> matmul_outer -> decrypt/decode)."""
import sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer
from tools.workloads import cfg_matmul
a, b = cfg_matmul(2)
eng = CkksEngine(config_params(2))
def step():
    return matmul_outer(eng, encode_left(eng, a, 64), encode_right(eng, b, 64)).decode(eng)
for _ in range(3): step()
torch.cuda.synchronize()
print(f"launches_before_steps={eng._lib.vr_launch_count()}", flush=True)
t0 = time.perf_counter()
for _ in range(5): step()
torch.cuda.synchronize()
print(f"e2e ms/step {1e3*(time.perf_counter()-t0)/5:.3f}")
