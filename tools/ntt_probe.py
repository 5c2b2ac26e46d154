"""Forward NTT throughput (bench.py's `ntt` line) for configs 2 and 4."""
import sys; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2512_18646_b200 import CkksEngine, config_params
from bench import bench_ntt, int_peaks
for cfg in (2, 4):
    eng = CkksEngine(config_params(cfg)); torch.cuda.set_stream(eng._stream)
    r = bench_ntt(eng, 6548.8, int_peaks(eng))
    print(cfg, {k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items() if k != 'int_roofline'}, round(r['int_roofline']['frac'], 4))
