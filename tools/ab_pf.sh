timeout 300 python tools/chain_probe.py 2>&1 | tail -1
timeout 300 python tools/e2e_profile.py 2>&1 | tail -1
python -c "
import sys, json; sys.path.insert(0, '.')
from bench import bench_cfg4, bench_cfg3
print(json.dumps(bench_cfg4(steps=2))[:140]); print(json.dumps(bench_cfg3())[:130])" 2>&1 | tail -2
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-extra > gpurun_out/bench_quick.log 2>&1; echo "bench rc=$?"; python tools/show_bench.py gpurun_out/bench_quick.log
