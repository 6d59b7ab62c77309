timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/exp8_tests.log 2>&1
timeout 600 python bench.py --config C5 --no-cpu-baseline > gpurun_out/exp8_c5.log 2>&1
timeout 600 python bench.py --config C5B --no-cpu-baseline > gpurun_out/exp8_c5b.log 2>&1
timeout 600 python bench.py --slices 0 --auto-T 1 --no-cpu-baseline > gpurun_out/exp8_auto1.log 2>&1
timeout 600 python bench.py --slices 0 --auto-T 0 --no-cpu-baseline > gpurun_out/exp8_auto0.log 2>&1
