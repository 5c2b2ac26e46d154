timeout 300 python tools/chain_probe.py 2>&1 | tail -1
python -c "
import sys, json; sys.path.insert(0, '.')
from bench import bench_cfg1, bench_cfg2_alg3, bench_cfg3
print(round(bench_cfg1()['value']), round(bench_cfg2_alg3()['value'], 1), round(bench_cfg3(steps=5)['value']))" 2>&1 | tail -1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
