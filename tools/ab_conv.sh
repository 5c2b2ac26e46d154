python -c "
import sys, json; sys.path.insert(0, '.')
from bench import bench_cfg4
print(json.dumps(bench_cfg4(steps=2))[:170])" 2>&1 | tail -1
python tools/step_profile.py --cfg 4 --steps 1 > gpurun_out/prof4_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k_conv_mac -s $(grep launches_before gpurun_out/prof4_plain.log | cut -d= -f2 | awk '{print 0}') -c 9 --csv --log-file gpurun_out/conv_metrics.csv python tools/step_profile.py --cfg 4 --steps 1 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 900 python -m pytest tests -q -m gpu -x -k "conv or cnn or cfg" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
