"""Host (Python + driver) time per matmul_outer call vs device time."""
import cProfile, pstats, sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer
from tools.workloads import cfg_matmul
a, b = cfg_matmul(2)
eng = CkksEngine(config_params(2))
L, R = encode_left(eng, a, 64), encode_right(eng, b, 64)
for _ in range(20): matmul_outer(eng, L, R)
torch.cuda.synchronize()
for steps in (10, 50, 200):
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); st.record(eng._stream)
    for _ in range(steps): matmul_outer(eng, L, R)
    t1 = time.perf_counter(); en.record(eng._stream); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"steps={steps}: host submit {1e3*(t1-t0)/steps:.3f} ms/step, device {st.elapsed_time(en)/steps:.3f} ms/step, wall {1e3*(t2-t0)/steps:.3f}")
pr = cProfile.Profile(); pr.enable()
for _ in range(100): matmul_outer(eng, L, R)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
# C-ABI call alone (pre-built pointer arrays): host cost of the C++ driver + its launches
from paper_2512_18646_b200 import _lib
lp = _lib.ptr_array([c.ptr() for c in L.cts]); rp = _lib.ptr_array([c.ptr() for c in R.cts])
outs = torch.empty((1, 2, eng.L, eng.N), dtype=torch.int64, device=eng.device); op = _lib.row_ptrs(outs, 1)
for _ in range(20): eng._lib.vr_matmul_outer(eng.handle, lp, rp, 64, 1, eng.L, op)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200): eng._lib.vr_matmul_outer(eng.handle, lp, rp, 64, 1, eng.L, op)
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"C-ABI vr_matmul_outer host submit {1e3*(t1-t0)/200:.3f} ms/call")
