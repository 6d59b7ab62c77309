set -x
M=sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,gpu__time_duration.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed
for v in default notma noepi; do
  if [ $v = default ]; then L=""; else L=$PWD/paper_2306_11975_b200/variants/libozimmu_$v.so; fi
  OZIMMU_LIB=$L timeout 300 ncu --kernel-name regex:k_oz_gemm --launch-skip 2 --launch-count 1 --clock-control none --metrics $M --csv python tools/stats_run.py 16384 9 > gpurun_out/exp1_ncu_$v.csv 2>&1
done
timeout 600 python tools/ab.py 16384 9 default paper_2306_11975_b200/variants/libozimmu_notma.so paper_2306_11975_b200/variants/libozimmu_noepi.so --rounds 2 > gpurun_out/exp1_ab.log 2>&1
