timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_zgemm.py tests/test_gpu_batched.py -x -q > gpurun_out/exp24_tests.log 2>&1
for i in 1 2; do timeout 300 python bench.py --steps 5 --no-e2e --no-cpu-baseline --no-cublas > gpurun_out/exp24_bench$i.log 2>&1; done
OZIMMU_SPLIT_NO_CLUSTER=1 timeout 300 python bench.py --steps 5 --no-e2e --no-cpu-baseline --no-cublas > gpurun_out/exp24_bench_nocl.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed
timeout 300 ncu --kernel-name regex:k_split --launch-skip 2 --launch-count 2 --clock-control none --metrics $M --csv python tools/stats_run.py 16384 9 > gpurun_out/exp24_ncu_split.csv 2>&1
