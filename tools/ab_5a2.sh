python tools/cfg5a_probe.py 2>&1 | tail -1
timeout 900 python -m pytest tests -q -m gpu -x -k "dist" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/bench_torchrun1.log 2>&1; echo "torchrun rc=$?"; python tools/show_bench.py gpurun_out/bench_torchrun1.log | grep cfg5
