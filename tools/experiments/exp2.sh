M=sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,gpu__time_duration.sum
for v in default ord0; do
  if [ $v = default ]; then L=""; else L=$PWD/paper_2306_11975_b200/variants/libozimmu_$v.so; fi
  OZIMMU_LIB=$L timeout 300 ncu --kernel-name regex:k_oz_gemm --launch-skip 2 --launch-count 1 --clock-control none --metrics $M --csv python tools/stats_run.py 16384 9 > gpurun_out/exp2_ncu_$v.csv 2>&1
done
OZIMMU_STATS=1 timeout 200 python tools/stats_run.py 16384 9 > gpurun_out/exp2_stats.log 2>&1
timeout 600 python tools/ab.py 16384 9 default paper_2306_11975_b200/variants/libozimmu_ord0.so --rounds 2 > gpurun_out/exp2_ab.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/exp2_parity.log 2>&1
