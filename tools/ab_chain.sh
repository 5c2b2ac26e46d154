for v in 1 2 4; do echo -n "VR_CHAIN_PER_SM=$v "; VR_CHAIN_PER_SM=$v timeout 300 python tools/chain_probe.py 2>&1 | tail -1; done
python tools/relin_probe.py > gpurun_out/rp.log 2>&1; S=$(grep launches_before gpurun_out/rp.log | cut -d= -f2)
ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum --clock-control none -s $S -c 6 --csv --log-file gpurun_out/launches_chain.csv python tools/relin_probe.py > /dev/null 2>&1; echo "ncu rc=$?"
