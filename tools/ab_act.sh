python -c "
import sys, json; sys.path.insert(0, '.')
from bench import bench_cfg4
print(json.dumps(bench_cfg4(steps=2))[:170])" 2>&1 | tail -1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
