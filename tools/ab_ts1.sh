for v in 0 1 2 4 5; do echo -n "VR_TS1_VARIANT=$v "; VR_TS1_VARIANT=$v timeout 300 python tools/chain_probe.py 2>&1 | tail -1; done
for v in 0 3; do echo -n "VR_TS2_VARIANT=$v "; VR_TS2_VARIANT=$v timeout 300 python tools/chain_probe.py 2>&1 | tail -1; done
