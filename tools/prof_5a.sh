for v in 0 1; do echo -n "VR_TS4=$v "; VR_TS4=$v python tools/cfg5a_probe.py 2>&1 | tail -1; done
timeout 900 python -m pytest tests -q -m gpu -x -k "cfg5 or dist or shard or matmul" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
