python tools/alg3_probe.py 2>&1 | tail -2
python -c "
import sys; sys.path.insert(0, '.')
import torch
from bench import bench_cfg2_alg3
r = bench_cfg2_alg3(steps=1)
print(r)
" 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_alg3.csv python -c "
import sys; sys.path.insert(0, '.')
from bench import bench_cfg2_alg3
bench_cfg2_alg3(steps=1)" > /dev/null 2>&1; echo "ncu rc=$?"
