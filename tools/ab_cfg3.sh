for ug in 1 2 3; do
S=$(VR_PMV_UG=$ug python tools/cfg3_profile.py 2>&1 | tee /dev/stderr | grep launches_before | cut -d= -f2)
VR_PMV_UG=$ug ncu --metrics gpu__time_duration.sum --clock-control none -s $S -c 100 --csv --log-file gpurun_out/launches_cfg3_$ug.csv python tools/cfg3_profile.py > /dev/null 2>&1; echo "ncu rc=$?"
done
