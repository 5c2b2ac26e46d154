"""Host cost of the pieces of CkksEngine.enc_strided (encode_left of cfg 2)."""
import sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left
from paper_2512_18646_b200 import _lib
from tools.workloads import cfg_matmul
a, b = cfg_matmul(2)
eng = CkksEngine(config_params(2))
for _ in range(5): encode_left(eng, a, 64)
torch.cuda.synchronize()
arr = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
T = {k: [] for k in ("h2d", "empty", "ctypes", "wrap", "full")}
for it in range(40):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); d = eng._h2d(arr)
    t1 = time.perf_counter(); out = eng._empty(1, eng.L, 64)
    t2 = time.perf_counter()
    _lib.check(eng._lib.vr_encrypt_strided(eng._h, d.data_ptr(), 1, 64, 0, 64, 4096, 64, eng.L, eng.scales[eng.L], 1000 + it * 64, out.data_ptr()))
    t3 = time.perf_counter(); w = [eng._wrap(out[i], eng.L, 0, None) for i in range(64)]
    t4 = time.perf_counter()
    torch.cuda.synchronize(); t5 = time.perf_counter(); encode_left(eng, a, 64); t6 = time.perf_counter()
    for k, v in zip(T, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t6 - t5)): T[k].append(v * 1e6)
print({k: round(float(np.median(v)), 1) for k, v in T.items()}, "us")
