timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/exp3_tests.log 2>&1
M=sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,gpu__time_duration.sum
OZIMMU_LIB= timeout 300 ncu --kernel-name regex:k_oz_gemm --launch-skip 2 --launch-count 1 --clock-control none --metrics $M --csv python tools/stats_run.py 16384 9 > gpurun_out/exp3_ncu.csv 2>&1
OZIMMU_STATS=1 timeout 200 python tools/stats_run.py 16384 9 > gpurun_out/exp3_stats.log 2>&1
timeout 600 python tools/ab.py 16384 9 default paper_2306_11975_b200/variants/libozimmu_ord0.so --rounds 2 > gpurun_out/exp3_ab.log 2>&1
