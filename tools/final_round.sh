bash tools/gpu_check.sh
bash tools/prof_ts.sh
# launch list of the bench command itself (headline path; cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-extra > gpurun_out/ncu_bench.log 2>&1; echo "ncu bench rc=$?"
python tools/cfg3_profile.py > gpurun_out/cfg3_plain.log 2>&1; S=$(grep launches_before gpurun_out/cfg3_plain.log | cut -d= -f2)
ncu --metrics gpu__time_duration.sum --clock-control none -s $S -c 300 --csv --log-file gpurun_out/launches_cfg3.csv python tools/cfg3_profile.py > /dev/null 2>&1; echo "ncu3 rc=$?"
python tools/cfg5a_prof.py > gpurun_out/p5.log 2>&1; S=$(grep launches_before gpurun_out/p5.log | cut -d= -f2)
ncu --metrics gpu__time_duration.sum --clock-control none -s $S -c 60 --csv --log-file gpurun_out/launches_5a.csv python tools/cfg5a_prof.py > /dev/null 2>&1; echo "ncu5a rc=$?"
