for cg in 1 2 4 8; do echo -n "CG=$cg: "; VR_KS_CG=$cg python tools/cfg4_hosttime.py 2>&1 | grep "iter [4-7]" | awk '{print $6}' | tr '\n' ' '; echo; done
