# usage: bash tools/run_ncu_full.sh <kernel-regex> <skip> <count> <tag> [step_profile args...]
K=$1; S=$2; C=$3; TAG=$4; shift 4
python tools/step_profile.py "$@" > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C -o gpurun_out/prof_$TAG python tools/step_profile.py "$@" > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu $TAG rc=$?"
