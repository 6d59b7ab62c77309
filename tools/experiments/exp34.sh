timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_batched.py tests/test_gpu_zgemm.py -x -q > gpurun_out/exp34_tests.log 2>&1
timeout 120 python tools/tiny_probe.py > gpurun_out/exp34_tiny.log 2>&1
OZIMMU_STATS=1 timeout 100 python tools/stats_run.py 1024 9 > gpurun_out/exp34_stats.log 2>&1
timeout 300 python tools/shape_probe.py > gpurun_out/exp34_shapes.log 2>&1
timeout 600 python tools/ab.py 16384 9 default --rounds 2 > gpurun_out/exp34_ab.log 2>&1
