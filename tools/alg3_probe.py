"""Config-2 Algorithm 3 (revolver matmul) device time per product, plus the top host functions."""
import cProfile, pstats, sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench

print(bench.bench_cfg2_alg3(steps=5))
pr = cProfile.Profile()
pr.enable()
bench.bench_cfg2_alg3(steps=2)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
