for v in 256 0; do echo "VR_NTT_CL=$v"; VR_NTT_CL=$v python tools/e2e_profile.py 2>&1 | tail -1; VR_NTT_CL=$v python tools/e2e_phases.py 2>&1 | tail -1; done
