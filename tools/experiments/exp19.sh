for cfg in "OZIMMU_B_STAGES=3 OZIMMU_CLUSTER=1" "OZIMMU_B_STAGES=3"; do
  for N in 8192 16384; do
  env $cfg timeout 60 python tools/quick_gemm.py $N 9 >> gpurun_out/exp19.log 2>&1 || echo "FAIL $cfg N=$N" >> gpurun_out/exp19.log
  done
done
env OZIMMU_A_STAGES=3 timeout 60 python tools/quick_gemm.py 16384 9 >> gpurun_out/exp19.log 2>&1 || echo "FAIL A3 16384" >> gpurun_out/exp19.log
