python tools/e2e_profile.py > gpurun_out/e2e_plain.log 2>&1; cat gpurun_out/e2e_plain.log | tail -1
S=$(grep launches_before gpurun_out/e2e_plain.log | cut -d= -f2)
ncu --metrics gpu__time_duration.sum --clock-control none -s $S -c 200 --csv --log-file gpurun_out/launches_e2e.csv python tools/e2e_profile.py > /dev/null 2>&1; echo "ncu rc=$?"
timeout 900 python -m pytest tests -q -m gpu -x -k "decode or dec or matmul or reference" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
