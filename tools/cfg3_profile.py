"""A few config-3 CNN passes (model encoded once) for ncu launch lists; prints wall time per pass."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2512_18646_b200 import CkksEngine, config_params
from paper_2512_18646_b200.cnn import cnn_cfg3, encode_cfg3_model
from tools.workloads import cfg3
imgs, w, w1, w2 = cfg3()
eng = CkksEngine(config_params(3))
model = encode_cfg3_model(eng, w, w1, w2)
for _ in range(2): cnn_cfg3(eng, imgs, w, model=model)
torch.cuda.synchronize()
print(f"launches_before_steps={eng._lib.vr_launch_count()}", flush=True)
t0 = time.perf_counter(); l0 = eng._lib.vr_launch_count()
for _ in range(3): cnn_cfg3(eng, imgs, w, model=model)
torch.cuda.synchronize()
print(f"wall ms/pass {1e3*(time.perf_counter()-t0)/3:.3f} launches/pass {(eng._lib.vr_launch_count()-l0)/3}")
