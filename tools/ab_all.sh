python tools/ntt_probe.py 2>&1 | cut -c1-200
python tools/chain_probe.py 2>&1 | tail -1
python tools/e2e_profile.py 2>&1 | tail -1
python -c "
import sys, json; sys.path.insert(0, '.')
from bench import bench_cfg4
print(json.dumps(bench_cfg4(steps=2)))" 2>&1 | tail -1 | cut -c1-200
