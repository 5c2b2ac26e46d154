for v in 0 64; do echo -n "VR_MODUP_COLS=$v "; VR_MODUP_COLS=$v timeout 300 python tools/chain_probe.py 2>&1 | tail -1; done
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
