"""Host submit vs device time of repeated matmul_outer calls (bench.py's device loop), per process."""
import sys, time; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer
from tools.workloads import cfg_matmul
a, b = cfg_matmul(2)
eng = CkksEngine(config_params(2))
L, R = encode_left(eng, a, 64), encode_right(eng, b, 64)
for _ in range(5): matmul_outer(eng, L, R)
torch.cuda.synchronize()
for rep in range(3):
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t0 = time.perf_counter(); st.record(eng._stream)
    for _ in range(200): matmul_outer(eng, L, R)
    t1 = time.perf_counter(); en.record(eng._stream); torch.cuda.synchronize()
    print(f"rep{rep}: host {1e3*(t1-t0)/200:.3f} ms/call  device {st.elapsed_time(en)/200:.3f} ms/call", flush=True)
