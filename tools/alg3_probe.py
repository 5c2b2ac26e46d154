import sys, json; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import bench_cfg2_alg3
print(json.dumps(bench_cfg2_alg3()))
