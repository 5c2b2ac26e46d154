timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
for v in 0 64 100000000; do echo "VR_NTT_SMALL=$v"; VR_NTT_SMALL=$v python tools/host_overhead.py 2>&1 | sed -n 3p; VR_NTT_SMALL=$v python tools/cfg4_hosttime.py 2>&1 | grep "iter 6" | awk '{print "cfg4", $6}'; done
