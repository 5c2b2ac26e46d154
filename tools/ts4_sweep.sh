for v in 0 1 2; do echo -n "variant $v: "; VR_TS_VARIANT=$v python tools/cfg5a_probe.py 2>&1 | tail -1; done
