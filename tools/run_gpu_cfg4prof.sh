timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_tests.log
python tools/step_profile.py --cfg 4 --steps 1 --images 16 --filters 16 > gpurun_out/prof4_plain.log 2>&1 && cat gpurun_out/prof4_plain.log && \
ncu --metrics gpu__time_duration.sum --clock-control none -s $(grep launches_before gpurun_out/prof4_plain.log | cut -d= -f2) -c 3000 --csv --log-file gpurun_out/launches_cfg4.csv python tools/step_profile.py --cfg 4 --steps 1 > gpurun_out/ncu4.log 2>&1; echo "ncu rc=$?"
