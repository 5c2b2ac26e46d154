import sys; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left
from tools.workloads import cfg_matmul
a, b = cfg_matmul(2)
eng = CkksEngine(config_params(2))
for _ in range(3):
    L = encode_left(eng, a, 64)
    eng.dec(L.cts[0])
torch.cuda.synchronize()
