python tools/step_profile.py --cfg 4 --steps 1 > /dev/null 2>&1
for e in 2; do
ncu --set full --clock-control none --import-source on -k regex:k_conv_mac -s 7 -c 1 -o /tmp/prof_conv$e python tools/step_profile.py --cfg 4 --steps 1 > gpurun_out/ncu_conv.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_conv$e.ncu-rep --page raw --csv > gpurun_out/conv_raw$e.csv 2>&1
ncu -i /tmp/prof_conv$e.ncu-rep --page source --csv --print-source sass > gpurun_out/conv_sass$e.csv 2>&1
done
