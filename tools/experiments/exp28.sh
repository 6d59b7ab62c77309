timeout 600 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/exp28_dist.log 2>&1
OZIMMU_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 2 --warmup 3 --config C3 --grid 2x2 --no-cpu-baseline > gpurun_out/exp28_bench4.log 2>&1
OZIMMU_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 2 --steps 2 --warmup 3 --config C3 --no-cpu-baseline > gpurun_out/exp28_bench2.log 2>&1
