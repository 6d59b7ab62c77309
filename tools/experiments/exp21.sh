for N in 4096 8192 16384 4096 8192; do
  OZIMMU_A_STAGES=3 timeout 60 python tools/quick_gemm.py $N 9 >> gpurun_out/exp21.log 2>&1 && echo "PASS A3 N=$N" >> gpurun_out/exp21.log || echo "FAIL A3 N=$N" >> gpurun_out/exp21.log
  OZIMMU_B_STAGES=3 timeout 60 python tools/quick_gemm.py $N 9 >> gpurun_out/exp21.log 2>&1 && echo "PASS B3 N=$N" >> gpurun_out/exp21.log || echo "FAIL B3 N=$N" >> gpurun_out/exp21.log
done
timeout 900 python tools/ab.py 16384 9 default default@OZIMMU_B_STAGES=3 --rounds 2 > gpurun_out/exp21_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cluster.py -x -q > gpurun_out/exp21_tests.log 2>&1
