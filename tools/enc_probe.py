"""Device time of encode_left (64 column encryptions, config 2) and of the whole e2e step pieces."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right

eng = CkksEngine(config_params(int(sys.argv[1]) if len(sys.argv) > 1 else 2))
a = np.random.default_rng(1).uniform(-1, 1, (64, 64))
dev = torch.from_numpy(a.reshape(-1)).cuda()
from paper_2512_18646_b200 import _lib
out = torch.empty((64, 2, eng.L + 1, eng.N), dtype=torch.int64, device="cuda")


def enc():
    _lib.check(eng._lib.vr_encrypt_strided(eng.handle, dev.data_ptr(), 1, 64, 0, 64, 4096, 64, eng.L, eng.scales[eng.L], 0,
                                           out.data_ptr()))


for _ in range(5):
    enc()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
st.record()
for _ in range(50):
    enc()
en.record()
torch.cuda.synchronize()
print(f"encrypt 64 cts: {st.elapsed_time(en) / 50 * 1e3:.1f} us")
