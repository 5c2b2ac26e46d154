python tools/cfg3_profile.py > gpurun_out/cfg3_plain.log 2>&1; cat gpurun_out/cfg3_plain.log | tail -2
S=$(grep launches_before gpurun_out/cfg3_plain.log | cut -d= -f2)
ncu --metrics gpu__time_duration.sum --clock-control none -s $S -c 600 --csv --log-file gpurun_out/launches_cfg3.csv python tools/cfg3_profile.py > /dev/null 2>&1; echo "ncu rc=$?"
