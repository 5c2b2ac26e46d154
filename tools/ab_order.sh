for o in 4 0 1 2; do echo -n "VR_MM_ORDER=$o "; VR_MM_ORDER=$o timeout 300 python tools/chain_probe.py 2>&1 | tail -1; done
for h in 1 0; do echo -n "VR_TS_HINT=$h "; VR_TS_HINT=$h timeout 300 python tools/chain_probe.py 2>&1 | tail -1; done
