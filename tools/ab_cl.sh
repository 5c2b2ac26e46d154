for r in 1 2; do for v in 128 64 32; do echo -n "VR_NTT_CL=$v cfg3 "; VR_NTT_CL=$v python -c "
import sys, json; sys.path.insert(0, '.')
from bench import bench_cfg3
print(round(bench_cfg3(steps=5)['value']))" 2>&1 | tail -1; done; done
for v in 128 64 32; do echo -n "VR_NTT_CL=$v "; VR_NTT_CL=$v timeout 300 python tools/chain_probe.py 2>&1 | tail -1; VR_NTT_CL=$v python tools/e2e_profile.py 2>&1 | tail -1; done
