timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_graph.py tests/test_gpu_host.py tests/test_gpu_auto.py tests/test_gpu_stress.py tests/test_gpu_shim.py -x -q > gpurun_out/exp36_tests.log 2>&1
timeout 120 python tools/tiny_probe.py > gpurun_out/exp36_tiny.log 2>&1
timeout 300 python tools/shape_probe.py > gpurun_out/exp36_shapes.log 2>&1
for i in 1 2; do timeout 300 python bench.py --steps 5 --no-e2e --no-cpu-baseline --no-cublas > gpurun_out/exp36_bench$i.log 2>&1; done
