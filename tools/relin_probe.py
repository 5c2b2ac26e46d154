"""cfg-2 relinearise+rescale of one ciphertext, a few times (for ncu launch lists)."""
import sys; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2512_18646_b200 import CkksEngine, config_params, _lib
eng = CkksEngine(config_params(2)); lib = eng._lib; lv = eng.L
d3 = torch.randint(0, 1 << 30, (1, 3, lv + 1, eng.N), dtype=torch.int64, device=eng.device)
out = torch.empty((1, 2, lv, eng.N), dtype=torch.int64, device=eng.device)
f = lambda: lib.vr_relin_rescale(eng.handle, _lib.row_ptrs(d3), _lib.row_ptrs(out), 1, lv)  # noqa: E731
for _ in range(3): f()
torch.cuda.synchronize()
print(f"launches_before_steps={lib.vr_launch_count()}", flush=True)
for _ in range(3): f()
torch.cuda.synchronize()
