python tools/e2e_profile.py > /dev/null 2>&1
ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"k_decode|k_encode" -s 6 -c 2 -o /tmp/prof_dec python tools/e2e_profile.py > gpurun_out/ncu_dec.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_dec.ncu-rep --page source --csv --print-source sass > gpurun_out/dec_sass.csv 2>&1
ncu -i /tmp/prof_dec.ncu-rep --page raw --csv > gpurun_out/dec_raw.csv 2>&1
