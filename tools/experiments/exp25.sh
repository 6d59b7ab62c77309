M=gpu__time_duration.sum,dram__bytes_read.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed
for c in 2 4 8; do
OZIMMU_SPLIT_CL=$c timeout 300 ncu --kernel-name regex:k_split_contig --launch-skip 1 --launch-count 1 --clock-control none --metrics $M --csv python tools/stats_run.py 16384 9 > gpurun_out/exp25_ncu_cl$c.csv 2>&1
done
for c in 2 4 8; do OZIMMU_SPLIT_CL=$c timeout 300 python bench.py --steps 5 --no-e2e --no-cpu-baseline --no-cublas > gpurun_out/exp25_bench_cl$c.log 2>&1; done
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "split or full_size" > gpurun_out/exp25_tests.log 2>&1
