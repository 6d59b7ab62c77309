timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/exp23_tests.log 2>&1
for cfg in "OZIMMU_A_STAGES=2" "OZIMMU_CLUSTER=1" "OZIMMU_CLUSTER=2" "OZIMMU_CLUSTER=4"; do
  env $cfg timeout 300 python tools/stress.py 8 >> gpurun_out/exp23_stress.log 2>&1 || echo "FAIL/TIMEOUT $cfg" >> gpurun_out/exp23_stress.log
done
