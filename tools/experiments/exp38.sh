L=$PWD/paper_2306_11975_b200/variants/libozimmu_prog.so
OZIMMU_LIB=$L timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_zgemm.py tests/test_gpu_batched.py tests/test_gpu_stress.py -x -q > gpurun_out/exp38_tests.log 2>&1
OZIMMU_LIB=$L OZIMMU_A_STAGES=2 timeout 300 python tools/stress.py 4 > gpurun_out/exp38_stress.log 2>&1
OZIMMU_LIB=$L timeout 120 python tools/tiny_probe.py > gpurun_out/exp38_tiny.log 2>&1
timeout 120 python tools/tiny_probe.py >> gpurun_out/exp38_tiny.log 2>&1
timeout 900 python tools/ab.py 16384 9 default $L --rounds 3 > gpurun_out/exp38_ab.log 2>&1
OZIMMU_LIB=$L OZIMMU_STATS=1 timeout 100 python tools/stats_run.py 16384 9 > gpurun_out/exp38_stats.log 2>&1
