import sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import bench_cfg5a
r = bench_cfg5a(1, 0, 0, lambda x: x, lambda: None, steps=10)
print(f"cfg5a {r['value']:.1f} matmul/s  {r['ms_per_matmul']:.3f} ms  err {r['max_abs_err']:.1e}")
