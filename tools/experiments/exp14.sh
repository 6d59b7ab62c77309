timeout 600 python -m pytest tests/test_gpu_host.py -x -q > gpurun_out/exp14_tests.log 2>&1
rm -f gpurun_out/exp7_host.log; bash tools/exp7.sh; cp gpurun_out/exp7_host.log gpurun_out/exp14_host.log
