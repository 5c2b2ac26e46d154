"""Table-1 CNN batches (model encoded once) for ncu launch lists; prints wall time and launches per batch."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from oracle.sim import table1_weights
from paper_2512_18646_b200 import EngineParams, Kernel, ModelWeights, SlotEngine, encode_model, forward_encoded, pack_batch
act1 = (-0.00015120704, 0.4610149, 2.0225089, -1.4511951)
act2 = (-1.5650465, -0.9943767, 1.6794522, 0.5350255)
kw, kb, f1w, f1b, f2w, f2b = table1_weights(7)
weights = ModelWeights([Kernel(kw[i], bias=float(kb[i])) for i in range(4)], f1w, f1b, f2w, f2b, act1, act2)
imgs = np.random.default_rng(8).uniform(0, 1, size=(32, 28, 28))
eng = SlotEngine(EngineParams(slots=32768, prime_bits=(60,) + (45,) * 13))
model = encode_model(eng, weights)
forward_encoded(eng, pack_batch(eng, imgs), model).decode(eng)
torch.cuda.synchronize()
print(f"launches_before_steps={eng._lib.vr_launch_count()}", flush=True)
t0 = time.perf_counter(); l0 = eng._lib.vr_launch_count()
forward_encoded(eng, pack_batch(eng, imgs), model).decode(eng)
torch.cuda.synchronize()
print(f"wall ms/batch {1e3*(time.perf_counter()-t0):.3f} launches/batch {eng._lib.vr_launch_count()-l0}")
