#!/bin/bash
# A/B of the cluster NTT (VR_NTT_CL) on the NTT probe, the e2e step and config 4
for v in 0 default; do
  if [ $v = default ]; then unset VR_NTT_CL; else export VR_NTT_CL=$v; fi
  echo "== VR_NTT_CL=$v"
  python tools/ntt_probe.py 2>&1 | cut -c1-200
  python tools/e2e_host.py 2>&1 | head -1
  python -c "
import sys, json; sys.path.insert(0, '.')
from bench import bench_cfg4
print(json.dumps(bench_cfg4(steps=2)))" 2>&1 | tail -1 | cut -c1-250
done
