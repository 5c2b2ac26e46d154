for v in "0 0" "4 0" "4 4"; do set -- $v; echo "== VR_RELIN_IP=$1 VR_RELIN_CL=$2"; VR_RELIN_IP=$1 VR_RELIN_CL=$2 python tools/chain_probe.py 2>&1 | tail -1
VR_RELIN_IP=$1 VR_RELIN_CL=$2 python tools/relin_probe.py > gpurun_out/rp.log 2>&1; S=$(grep launches_before gpurun_out/rp.log | cut -d= -f2)
VR_RELIN_IP=$1 VR_RELIN_CL=$2 ncu --metrics gpu__time_duration.sum --clock-control none -s $S -c 40 --csv --log-file gpurun_out/launches_relin_$1_$2.csv python tools/relin_probe.py > /dev/null 2>&1; echo "ncu rc=$?"
done
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-extra > gpurun_out/bench_quick.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/bench_quick.log | cut -c1-400
