python tools/relin_probe.py > gpurun_out/rp.log 2>&1; S=$(grep launches_before gpurun_out/rp.log | cut -d= -f2)
VR_PDL=0 ncu --set full --clock-control none --import-source on -s $S -c ${NK:-9} -o /tmp/prof_relin python tools/relin_probe.py > gpurun_out/ncu_relin.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_relin.ncu-rep --page details --csv > gpurun_out/relin_details.csv 2>&1
ncu -i /tmp/prof_relin.ncu-rep --page raw --csv > gpurun_out/relin_raw.csv 2>&1
ls -la gpurun_out
