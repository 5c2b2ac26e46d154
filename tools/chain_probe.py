"""Device time of the cfg-2 matmul pieces: d2 sum, (d0,d1) sum, relin+rescale chain, whole matmul_outer."""
import sys; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch, numpy as np
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer, _lib
from tools.workloads import cfg_matmul
a, b = cfg_matmul(2)
eng = CkksEngine(config_params(2)); lib = eng._lib
L, R = encode_left(eng, a, 64), encode_right(eng, b, 64)
lp = _lib.ptr_array([c.ptr() for c in L.cts]); rp = _lib.ptr_array([c.ptr() for c in R.cts])
lv = eng.L
d3 = torch.empty((1, 3, lv + 1, eng.N), dtype=torch.int64, device=eng.device)
out = torch.empty((1, 2, lv, eng.N), dtype=torch.int64, device=eng.device)
def timeit(f, n=200):
    for _ in range(5): f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record(eng._stream)
    for _ in range(n): f()
    e.record(eng._stream); torch.cuda.synchronize(); return s.elapsed_time(e) / n * 1e3
res = {
 "d2_only": timeit(lambda: lib.vr_tensor_sum_mode(eng.handle, lp, rp, 64, lv, d3.data_ptr(), 1)),
 "d01_only": timeit(lambda: lib.vr_tensor_sum_mode(eng.handle, lp, rp, 64, lv, d3.data_ptr(), 2)),
 "all3": timeit(lambda: lib.vr_tensor_sum(eng.handle, lp, rp, 64, 1, lv, _lib.row_ptrs(d3))),
 "relin_rescale": timeit(lambda: lib.vr_relin_rescale(eng.handle, _lib.row_ptrs(d3), _lib.row_ptrs(out), 1, lv)),
 "matmul_outer": timeit(lambda: matmul_outer(eng, L, R)),
}
print({k: round(v, 1) for k, v in res.items()}, "us")
