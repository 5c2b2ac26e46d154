for v in 0 1 2 3 4 5 6 7; do echo -n "variant $v: "; VR_TS_VARIANT=$v python tools/bw_probe.py 2>&1 | grep k_tensor_sum; done
