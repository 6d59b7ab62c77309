for N in 4096 8192 16384; do
  for cfg in "OZIMMU_A_STAGES=3" "OZIMMU_B_STAGES=3" "OZIMMU_CLUSTER=2"; do
    env $cfg timeout 60 python tools/quick_gemm.py $N 9 >> gpurun_out/exp22.log 2>&1 && echo "PASS $cfg N=$N" >> gpurun_out/exp22.log || echo "FAIL $cfg N=$N" >> gpurun_out/exp22.log
  done
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cluster.py -x -q > gpurun_out/exp22_tests.log 2>&1
timeout 500 python tools/ab.py 16384 9 default default@OZIMMU_B_STAGES=3 --rounds 2 > gpurun_out/exp22_ab.log 2>&1
