timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/bench_torchrun1.log 2>&1; echo "torchrun rc=$?"
python tools/show_bench.py gpurun_out/bench_torchrun1.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/bench_ref_torchrun1.log 2>&1; echo "ref torchrun rc=$?"; tail -c 300 gpurun_out/bench_ref_torchrun1.log
nproc; lscpu | grep "Model name"
