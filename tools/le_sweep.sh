for le in 3 4; do echo "VR_NTT_BIG_LE=$le"; VR_NTT_BIG_LE=$le python tools/ntt_probe.py 2>&1 | cut -c1-200; VR_NTT_BIG_LE=$le python tools/cfg4_hosttime.py 2>&1 | grep "iter 6" | awk '{print "cfg4", $6}'; done
VR_NTT_BIG_LE=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
