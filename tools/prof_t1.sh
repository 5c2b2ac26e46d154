python tools/t1_profile.py > gpurun_out/t1_plain.log 2>&1; tail -1 gpurun_out/t1_plain.log
S=$(grep launches_before gpurun_out/t1_plain.log | cut -d= -f2)
ncu --metrics gpu__time_duration.sum --clock-control none -s $S -c 9000 --csv --log-file gpurun_out/launches_t1.csv python tools/t1_profile.py > /dev/null 2>&1; echo "ncu rc=$?"
