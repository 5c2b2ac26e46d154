for v in 0 1; do echo -n "SKIP01=$v split0 "; VR_DBG_SKIP01=$v VR_MM_SPLIT=0 python tools/chain_probe.py 2>&1 | tail -1; done
