timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
python tools/step_profile.py --cfg 2 --steps 3 > gpurun_out/prof_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s $(grep launches_before gpurun_out/prof_plain.log | cut -d= -f2) -c 40 --csv --log-file gpurun_out/launches_cfg2.csv python tools/step_profile.py --cfg 2 --steps 3 > gpurun_out/ncu_launch.log 2>&1; echo "ncu2 rc=$?"
python tools/step_profile.py --cfg 4 --steps 1 > gpurun_out/prof4_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s $(grep launches_before gpurun_out/prof4_plain.log | cut -d= -f2) -c 2000 --csv --log-file gpurun_out/launches_cfg4.csv python tools/step_profile.py --cfg 4 --steps 1 > gpurun_out/ncu4.log 2>&1; echo "ncu4 rc=$?"
bash tools/run_ncu_full.sh "k_tensor_sum" 0 2 ts --cfg 2 --steps 2
