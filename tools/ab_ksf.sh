for v in 0 8; do echo "VR_KS_FUSED_MIN=$v"; VR_KS_FUSED_MIN=$v python -c "
import sys, json; sys.path.insert(0, '.')
from bench import bench_cfg4, bench_cfg3
print(json.dumps(bench_cfg4(steps=2))[:160]); print(json.dumps(bench_cfg3())[:150])" 2>&1 | tail -2
VR_KS_FUSED_MIN=$v python tools/t1_profile.py 2>&1 | tail -1; done
timeout 900 python -m pytest tests -q -m gpu -x -k "cnn or cfg or relin or mul" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
