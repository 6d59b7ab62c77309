timeout 600 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/exp9_dist.log 2>&1
OZIMMU_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --config C3 > gpurun_out/exp9_bench2.log 2>&1
for b in 2 4 8 16; do OZIMMU_SPLIT_BPS=$b timeout 300 python bench.py --steps 5 --no-e2e --no-cpu-baseline --no-cublas > gpurun_out/exp9_bps$b.log 2>&1; done
