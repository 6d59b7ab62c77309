timeout 900 python tools/ab.py 16384 9 default default@OZIMMU_WAVE_LAG=1 default@OZIMMU_WAVE_LAG=2 --rounds 2 > gpurun_out/exp31_ab.log 2>&1
OZIMMU_STATS=1 OZIMMU_WAVE_LAG=1 timeout 200 python tools/stats_run.py 16384 9 > gpurun_out/exp31_stats.log 2>&1
M=dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
OZIMMU_WAVE_LAG=1 timeout 300 ncu --kernel-name regex:k_oz_gemm --launch-skip 2 --launch-count 1 --clock-control none --metrics $M --csv python tools/stats_run.py 16384 9 > gpurun_out/exp31_ncu.csv 2>&1
