for cg in 1 2 4; do echo "VR_KS_CG=$cg"; VR_KS_CG=$cg python tools/t1_profile.py 2>&1 | tail -1
VR_KS_CG=$cg python -c "
import sys, json; sys.path.insert(0, '.')
from bench import bench_cfg4
print(json.dumps(bench_cfg4(steps=2)))" 2>&1 | tail -1 | cut -c1-150; done
