import sys, json; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import bench_table1
print(json.dumps(bench_table1()))
