TAG=${1:-r02e}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_split_fused.py tests/test_gpu_parity.py tests/test_gpu_zgemm.py tests/test_gpu_fuzz.py tests/test_gpu_batched.py tests/test_gpu_bigk.py tests/test_gpu_streamk.py tests/test_gpu_cluster.py tests/test_gpu_stress.py -q -x > gpurun_out/${TAG}_tests.log 2>&1
tail -3 gpurun_out/${TAG}_tests.log
for b in 2 4 16; do OZIMMU_SPLIT_BPS=$b python tools/split_bench.py --sizes 16384,2048 | sed "s/^/bps$b /"; done > gpurun_out/${TAG}_split.txt 2>&1
for b in 2 3; do OZIMMU_SPLIT_FUSED=1 OZIMMU_SPLIT_FUSED_BPS=$b python tools/split_bench.py --sizes 16384 | sed "s/^/fused_bps$b /"; done >> gpurun_out/${TAG}_split.txt 2>&1
cat gpurun_out/${TAG}_split.txt
C5_DS=8,10 C5_SS=8 C5_IT=3 timeout 300 python tools/c5_sweep.py > gpurun_out/${TAG}_c5.jsonl 2>&1
OZIMMU_ACC2=0 C5_DS=8,10 C5_SS=8 C5_IT=3 timeout 300 python tools/c5_sweep.py | sed "s/^/acc1 /" >> gpurun_out/${TAG}_c5.jsonl 2>&1
cat gpurun_out/${TAG}_c5.jsonl
timeout 300 python tools/small_shapes.py > gpurun_out/${TAG}_small.jsonl 2>&1
cat gpurun_out/${TAG}_small.jsonl
