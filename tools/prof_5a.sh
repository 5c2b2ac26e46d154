for v in 0 2 3 4; do echo -n "VR_TS4=$v "; VR_TS4=$v python tools/cfg5a_probe.py 2>&1 | tail -1; done
VR_TS4=2 timeout 900 python -m pytest tests -q -m gpu -x -k "dist or matmul_outer_blocks or blocks" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
