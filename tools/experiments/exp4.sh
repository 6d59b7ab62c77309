timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cluster.py -x -q > gpurun_out/exp4_tests.log 2>&1
M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for v in default nosnake; do
  if [ $v = default ]; then L=""; else L=$PWD/paper_2306_11975_b200/variants/libozimmu_$v.so; fi
  OZIMMU_LIB=$L timeout 300 ncu --kernel-name regex:k_oz_gemm --launch-skip 2 --launch-count 1 --clock-control none --metrics $M --csv python tools/stats_run.py 16384 9 > gpurun_out/exp4_ncu_$v.csv 2>&1
done
timeout 900 python tools/ab.py 16384 9 default paper_2306_11975_b200/variants/libozimmu_nosnake.so default@OZIMMU_CLUSTER=2 --rounds 2 > gpurun_out/exp4_ab.log 2>&1
timeout 300 python tools/int8_peak.py 16384 > gpurun_out/exp4_int8_peak.log 2>&1
