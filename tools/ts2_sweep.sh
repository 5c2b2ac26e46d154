for v in 0 3 8 9 10; do echo -n "ts2 variant $v: "; VR_TS2_VARIANT=$v python tools/chain_probe.py 2>&1 | tail -1; done
for v in 0 1 2 3 4 5 6 7; do echo -n "ts1 variant $v: "; VR_TS2_VARIANT=3 VR_TS1_VARIANT=$v python tools/chain_probe.py 2>&1 | tail -1; done
