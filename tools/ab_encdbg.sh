for v in 0 1; do
VR_DBG_ENC=$v python tools/e2e_profile.py > gpurun_out/e2e_plain.log 2>&1; S=$(grep launches_before gpurun_out/e2e_plain.log | cut -d= -f2)
VR_DBG_ENC=$v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ntt_cl8 -c 8 --csv --log-file gpurun_out/enc_dbg_$v.csv python tools/e2e_profile.py > /dev/null 2>&1; echo "ncu $v rc=$?"
done
