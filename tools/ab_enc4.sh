for v in 0 1; do echo "VR_ENC_R4=$v"; VR_ENC_R4=$v python tools/e2e_profile.py > gpurun_out/e2e_plain.log 2>&1; tail -1 gpurun_out/e2e_plain.log
S=$(grep launches_before gpurun_out/e2e_plain.log | cut -d= -f2)
VR_ENC_R4=$v ncu --metrics gpu__time_duration.sum --clock-control none -s $S -c 200 --csv --log-file gpurun_out/launches_e2e_$v.csv python tools/e2e_profile.py > /dev/null 2>&1; done
VR_ENC_R4=1 timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
