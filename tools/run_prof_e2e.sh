# e2e cfg-2 step: launch list + ncu --set full of the fused encryption NTT, the slot FFTs
python tools/e2e_profile.py > gpurun_out/e2e_plain.log 2>&1; echo "e2e plain rc=$?"; cat gpurun_out/e2e_plain.log
S=$(grep launches_before gpurun_out/e2e_plain.log | cut -d= -f2)
ncu --metrics gpu__time_duration.sum --clock-control none -s $S -c 200 --csv --log-file gpurun_out/launches_e2e.csv python tools/e2e_profile.py > gpurun_out/ncu_e2e_launch.log 2>&1; echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"ntt_cl8|k_encode|k_decode" -s 12 -c 4 -o gpurun_out/prof_enc python tools/e2e_profile.py > gpurun_out/ncu_enc.log 2>&1; echo "ncu full rc=$?"
python tools/step_profile.py --cfg 2 --steps 3 > gpurun_out/prof_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s $(grep launches_before gpurun_out/prof_plain.log | cut -d= -f2) -c 40 --csv --log-file gpurun_out/launches_cfg2.csv python tools/step_profile.py --cfg 2 --steps 3 > gpurun_out/ncu_launch.log 2>&1; echo "ncu2 rc=$?"
