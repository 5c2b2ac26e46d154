for v in 32 24; do for r in 1 2; do echo -n "VR_NTT_CL=$v "; VR_NTT_CL=$v python -c "
import sys, json; sys.path.insert(0, '.')
from bench import bench_cfg1, bench_cfg2_alg3
print(round(bench_cfg1()['value']), round(bench_cfg2_alg3()['value'], 1))" 2>&1 | tail -1; done; done
