# slicing check: parity of the slicing paths, split bench (fused vs two-launch), ncu of the
# fused kernel, plus probes (C5 d=8 phases, small shapes with stall counters)
TAG=${1:-r02c}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_split_fused.py tests/test_gpu_parity.py tests/test_gpu_zgemm.py tests/test_gpu_fuzz.py tests/test_gpu_batched.py tests/test_gpu_bigk.py -q -x > gpurun_out/${TAG}_tests.log 2>&1
tail -3 gpurun_out/${TAG}_tests.log
python tools/split_bench.py > gpurun_out/${TAG}_split_fused.jsonl 2>&1
OZIMMU_SPLIT_FUSED=0 python tools/split_bench.py --sizes 16384,2048 > gpurun_out/${TAG}_split_old.jsonl 2>&1
cat gpurun_out/${TAG}_split_fused.jsonl gpurun_out/${TAG}_split_old.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_split_fused -s 6 -c 2 -o gpurun_out/prof_split_${TAG} python tools/split_bench.py --sizes 16384 --it 3 > gpurun_out/ncu_split_${TAG}.log 2>&1
echo ncu rc=$?
C5_DS=8 C5_SS=8 C5_IT=3 timeout 300 python tools/c5_sweep.py > gpurun_out/${TAG}_c5d8.jsonl 2>&1
cat gpurun_out/${TAG}_c5d8.jsonl
OZIMMU_STATS=1 timeout 300 python tools/small_shapes.py --quick --shapes 1024,2048 > gpurun_out/${TAG}_small_stats.log 2>&1
timeout 300 python tools/small_shapes.py > gpurun_out/${TAG}_small.jsonl 2>&1
cat gpurun_out/${TAG}_small.jsonl
