python tools/step_profile.py --cfg 2 --steps 2 > gpurun_out/plain_ts.log 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:k_tensor_sum -s 0 -c 2 -o /tmp/prof_ts python tools/step_profile.py --cfg 2 --steps 2 > gpurun_out/ncu_ts.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summarize.py /tmp/prof_ts.ncu-rep gpurun_out/ncu_summary.json
ncu -i /tmp/prof_ts.ncu-rep --page raw --csv > gpurun_out/ts_raw.csv 2>&1
python tools/step_profile.py --cfg 2 --steps 3 > gpurun_out/prof_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s $(grep launches_before gpurun_out/prof_plain.log | cut -d= -f2) -c 40 --csv --log-file gpurun_out/launches_cfg2.csv python tools/step_profile.py --cfg 2 --steps 3 > gpurun_out/ncu_launch.log 2>&1; echo "ncu2 rc=$?"
python tools/e2e_profile.py > gpurun_out/e2e_plain.log 2>&1; S=$(grep launches_before gpurun_out/e2e_plain.log | cut -d= -f2)
ncu --metrics gpu__time_duration.sum --clock-control none -s $S -c 200 --csv --log-file gpurun_out/launches_e2e.csv python tools/e2e_profile.py > gpurun_out/ncu_e2e_launch.log 2>&1; echo "ncu e2e rc=$?"
python tools/step_profile.py --cfg 4 --steps 1 > gpurun_out/prof4_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s $(grep launches_before gpurun_out/prof4_plain.log | cut -d= -f2) -c 2000 --csv --log-file gpurun_out/launches_cfg4.csv python tools/step_profile.py --cfg 4 --steps 1 > gpurun_out/ncu4.log 2>&1; echo "ncu4 rc=$?"
