timeout 120 ./tools/mma_bench > gpurun_out/exp6_mma.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_zgemm.py -x -q > gpurun_out/exp6_tests.log 2>&1
M=sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,gpu__time_duration.sum
timeout 300 ncu --kernel-name regex:k_oz_gemm --launch-skip 2 --launch-count 1 --clock-control none --metrics $M --csv python tools/stats_run.py 16384 9 > gpurun_out/exp6_ncu.csv 2>&1
timeout 900 python tools/ab.py 16384 9 default paper_2306_11975_b200/variants/libozimmu_prevbal.so --rounds 2 > gpurun_out/exp6_ab.log 2>&1
