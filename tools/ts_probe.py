"""Config-2 one-pass tensor sum (vr_tensor_sum, nb = 1) timed alone: GB/s of algorithmic bytes.
VR_TS_HINT=9 makes the consumers skip the arithmetic (stream-only diagnostic; results invalid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2512_18646_b200 import CkksEngine, _lib, config_params, encode_left, encode_right

eng = CkksEngine(config_params(2))
a, b = np.random.default_rng(1).uniform(-1, 1, (2, 64, 64))
L, R = encode_left(eng, a, 64), encode_right(eng, b, 64)
lp, rp = _lib.ptr_array([c.ptr() for c in L.cts]), _lib.ptr_array([c.ptr() for c in R.cts])
d3 = torch.empty((3, eng.L + 1, eng.N), dtype=torch.int64, device="cuda")
op = _lib.ptr_array([d3.data_ptr()])
f = lambda: _lib.check(eng._lib.vr_tensor_sum(eng.handle, lp, rp, 64, 1, eng.L, op))  # noqa: E731
for _ in range(5):
    f()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
st.record()
for _ in range(50):
    f()
en.record()
torch.cuda.synchronize()
t = st.elapsed_time(en) / 50 * 1e3
nb = 4 * 64 * 5 * eng.N * 8 + 3 * 5 * eng.N * 8
print(f"tensor sum: {t:.1f} us = {nb / t / 1e3:.0f} GB/s")
