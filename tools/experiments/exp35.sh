timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > gpurun_out/exp35_tests.log 2>&1
timeout 120 python tools/tiny_probe.py > gpurun_out/exp35_tiny.log 2>&1
OZIMMU_STATS=1 timeout 100 python tools/stats_run.py 1024 9 > gpurun_out/exp35_stats.log 2>&1
OZIMMU_STATS=1 timeout 100 python tools/stats_run.py 16384 9 >> gpurun_out/exp35_stats.log 2>&1
timeout 600 python tools/ab.py 16384 9 default --rounds 2 > gpurun_out/exp35_ab.log 2>&1
