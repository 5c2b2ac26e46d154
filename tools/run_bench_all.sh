timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 --no-extra > gpurun_out/bench_torchrun1.log 2>&1; echo "torchrun rc=$?"
nproc; lscpu | grep "Model name"
