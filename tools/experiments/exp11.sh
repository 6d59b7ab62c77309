M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for v in default hint1 hint2; do
  if [ $v = default ]; then L=""; else L=$PWD/paper_2306_11975_b200/variants/libozimmu_$v.so; fi
  OZIMMU_LIB=$L timeout 300 ncu --kernel-name regex:k_oz_gemm --launch-skip 2 --launch-count 1 --clock-control none --metrics $M --csv python tools/stats_run.py 16384 9 > gpurun_out/exp11_ncu_$v.csv 2>&1
done
timeout 900 python tools/ab.py 16384 9 default paper_2306_11975_b200/variants/libozimmu_hint1.so paper_2306_11975_b200/variants/libozimmu_hint2.so --rounds 2 > gpurun_out/exp11_ab.log 2>&1
