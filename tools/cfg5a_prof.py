"""cfg5a (1 GPU): a few sharded matmuls for ncu launch lists."""
import sys; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2512_18646_b200 import CkksEngine, config_params
from paper_2512_18646_b200.dist import encode_operands_sharded, matmul_outer_sharded
from tools.workloads import cfg_matmul
a, b = cfg_matmul(5)
blocks = [a[64 * i: 64 * (i + 1)] for i in range(4)]
eng = CkksEngine(config_params(5))
lefts, right = encode_operands_sharded(eng, blocks, b, 0, 256)
for _ in range(2): matmul_outer_sharded(eng, lefts, right)
torch.cuda.synchronize()
print(f"launches_before_steps={eng._lib.vr_launch_count()}", flush=True)
for _ in range(2): matmul_outer_sharded(eng, lefts, right)
torch.cuda.synchronize()
