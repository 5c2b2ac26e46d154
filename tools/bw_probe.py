"""Read-bandwidth probes: torch sum/copy over the 168 MB operand set vs k_tensor_sum."""
import sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, _lib
from tools.workloads import cfg_matmul

def timeit(fn, reps=20):
    for _ in range(3): fn()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); st.record()
    for _ in range(reps): fn()
    en.record(); torch.cuda.synchronize()
    return st.elapsed_time(en) / reps / 1e3

x = torch.randint(0, 2**40, (168 * 2**20 // 8,), dtype=torch.int64, device="cuda")
y = torch.empty_like(x)
t = timeit(lambda: x.sum()); print(f"torch int64 sum  168MB: {x.numel()*8/t/1e9:8.1f} GB/s read")
t = timeit(lambda: y.copy_(x)); print(f"torch copy       168MB: {2*x.numel()*8/t/1e9:8.1f} GB/s r+w")
xf = x.view(torch.float64)
t = timeit(lambda: xf.sum()); print(f"torch f64 sum    168MB: {x.numel()*8/t/1e9:8.1f} GB/s read")
big = torch.empty(2**31 // 8 * 4, dtype=torch.int64, device="cuda"); big2 = torch.empty_like(big)
t = timeit(lambda: big2.copy_(big), 10); print(f"torch copy 1 GiB       : {2*big.numel()*8/t/1e9:8.1f} GB/s r+w")
del big, big2
a, b = cfg_matmul(2)
eng = CkksEngine(config_params(2))
L, R = encode_left(eng, a, 64), encode_right(eng, b, 64)
lib = eng._lib
d3 = torch.empty((3, 5, eng.N), dtype=torch.int64, device="cuda")
pl = _lib.ptr_array([c.ptr() for c in L.cts]); pr = _lib.ptr_array([c.ptr() for c in R.cts]); po = _lib.ptr_array([d3.data_ptr()])
def ts(): _lib.check(lib.vr_tensor_sum(eng.handle, pl, pr, 64, 1, 4, po))
torch.cuda.set_stream(eng._stream)
t = timeit(ts); print(f"k_tensor_sum: {t*1e6:.1f} us, {169738240/t/1e9:.1f} GB/s")
