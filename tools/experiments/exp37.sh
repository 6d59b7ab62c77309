timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_zgemm.py tests/test_gpu_batched.py tests/test_gpu_host.py tests/test_gpu_stress.py -x -q > gpurun_out/exp37_tests.log 2>&1
timeout 120 python tools/tiny_probe.py > gpurun_out/exp37_tiny.log 2>&1
timeout 300 python tools/shape_probe.py > gpurun_out/exp37_shapes.log 2>&1
