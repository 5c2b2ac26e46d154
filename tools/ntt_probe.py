import sys; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2512_18646_b200 import CkksEngine, config_params
from bench import bench_ntt
for cfg in (2, 4):
    eng = CkksEngine(config_params(cfg)); torch.cuda.set_stream(eng._stream)
    r = bench_ntt(eng, 6553.3); print(cfg, {k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items() if k != 'int_roofline'}, r['int_roofline'])
