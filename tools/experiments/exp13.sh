timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_parity.py -x -q > gpurun_out/exp13_tests.log 2>&1
timeout 900 python tools/ab.py 16384 9 default default@OZIMMU_CLUSTER=4 default@OZIMMU_CLUSTER=1 --rounds 2 > gpurun_out/exp13_ab.log 2>&1
