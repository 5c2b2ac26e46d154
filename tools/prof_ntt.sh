for cfg in 2 4; do
ncu --set full --clock-control none --import-source on -k regex:"ntt_" -s 4 -c 4 -o /tmp/prof_ntt$cfg python tools/ntt_only.py $cfg > gpurun_out/ncu_ntt$cfg.log 2>&1; echo "ncu $cfg rc=$?"
ncu -i /tmp/prof_ntt$cfg.ncu-rep --page raw --csv > gpurun_out/ntt${cfg}_raw.csv 2>&1
ncu -i /tmp/prof_ntt$cfg.ncu-rep --page source --csv --print-source sass > gpurun_out/ntt${cfg}_sass.csv 2>&1
done
python tools/ntt_probe.py
ls -la gpurun_out
