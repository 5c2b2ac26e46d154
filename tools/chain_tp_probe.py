"""Throughput of the relinearise+rescale chain alone under the asynchronous slots: matmul_outer with
n = 1 column pair (the tensor sum is trivial), cfg-2 parameters; and with n = 64 for comparison."""
import sys, time; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer
eng = CkksEngine(config_params(2))
rng = np.random.default_rng(0)
for n in (1, 2, 8, 64):
    a, b = rng.uniform(-1, 1, (64, n)), rng.uniform(-1, 1, (n, 64))
    L, R = encode_left(eng, a, 64), encode_right(eng, b, 64)
    for _ in range(40): out = matmul_outer(eng, L, R)
    eng.join(); torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); st.record()
    for _ in range(400): out = matmul_outer(eng, L, R)
    host = (time.perf_counter() - t0) / 400 * 1e6
    eng.join(); en.record(); torch.cuda.synchronize()
    print(f"n={n:3d}: {st.elapsed_time(en) / 400 * 1e3:.1f} us per product (host {host:.1f} us per call), err {np.max(np.abs(out.decode(eng) - a @ b)):.1e}")
