"""A few forward NTTs (cfg-2: 1280 limbs at N=2^14 -> cluster kernel; cfg-4: 2048 limbs at N=2^15 -> two passes) for ncu."""
import sys; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2512_18646_b200 import CkksEngine, config_params
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
eng = CkksEngine(config_params(cfg))
data = torch.randint(0, 2 ** 39, (256, eng.L + 1, eng.N), dtype=torch.int64, device="cuda")
for _ in range(4):
    eng._lib.vr_ntt(eng.handle, data.data_ptr(), 256, eng.L + 1, 0, 0)
    eng._lib.vr_ntt(eng.handle, data.data_ptr(), 256, eng.L + 1, 0, 1)
torch.cuda.synchronize()
