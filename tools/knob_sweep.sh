for v in 64 16 128 512; do echo -n "VR_NTT_SMALL=$v "; VR_NTT_SMALL=$v timeout 300 python tools/chain_probe.py 2>&1 | tail -1; done
for v in 256 128 512 1024; do echo -n "VR_NTT_CL=$v "; VR_NTT_CL=$v timeout 300 python tools/e2e_profile.py 2>&1 | tail -1; done
for v in 256 128; do echo -n "VR_NTT_CL=$v cfg3 "; VR_NTT_CL=$v python -c "
import sys, json; sys.path.insert(0, '.')
from bench import bench_cfg3
print(json.dumps(bench_cfg3())[:130])" 2>&1 | tail -1; done
