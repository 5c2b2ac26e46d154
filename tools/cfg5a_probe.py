"""Config 5a on one GPU: device time of the 4-block tensor sum alone and of the whole sharded
matmul (matmul_outer_sharded_owned at world 1).  python tools/cfg5a_probe.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2512_18646_b200 import CkksEngine, _lib, config_params
from paper_2512_18646_b200.dist import encode_operands_sharded, matmul_outer_sharded_owned
from tools.workloads import cfg_matmul


def timed(fn, reps):
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    st.record()
    for _ in range(reps):
        fn()
    eng.join()
    en.record()
    torch.cuda.synchronize()
    return st.elapsed_time(en) / reps * 1e3


a, b = cfg_matmul(5)
blocks = [a[64 * i: 64 * (i + 1)] for i in range(4)]
eng = CkksEngine(config_params(5))
ls, r = encode_operands_sharded(eng, blocks, b, 0, 256)
lv = eng.L
part = torch.empty((4, 3, lv + 1, eng.N), dtype=torch.int64, device="cuda")
lp = _lib.ptr_array([c.ptr() for lf in ls for c in lf.cts])
rp = _lib.ptr_array([c.ptr() for c in r.cts])
op = _lib.row_ptrs(part, 4)
t_ts = timed(lambda: _lib.check(eng._lib.vr_tensor_sum(eng.handle, lp, rp, 256, 4, lv, op)), 10)
nbytes = (4 * 256 + 256) * 2 * (lv + 1) * eng.N * 8 + 4 * 3 * (lv + 1) * eng.N * 8
t_mm = timed(lambda: matmul_outer_sharded_owned(eng, ls, r), 5)
outs = matmul_outer_sharded_owned(eng, ls, r)
err = max(float(np.max(np.abs(eng.dec(o)[: 64 * 256].reshape(64, 256) - blocks[bi] @ b))) for bi, o in outs.items())
print(f"tensor_sum nb=4: {t_ts:.1f} us = {nbytes / t_ts / 1e3:.0f} GB/s (alg bytes {nbytes / 1e9:.2f} GB); "
      f"matmul: {t_mm:.1f} us = {1e6 / t_mm:.1f} HE matmul/s; max err {err:.2e}")
