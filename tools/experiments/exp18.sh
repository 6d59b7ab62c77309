for cfg in "OZIMMU_B_STAGES=3 OZIMMU_CLUSTER=1" "OZIMMU_B_STAGES=3" "OZIMMU_A_STAGES=3" "OZIMMU_A_STAGES=4" "OZIMMU_A_STAGES=5" "OZIMMU_CLUSTER=1 OZIMMU_A_STAGES=3"; do
  env $cfg timeout 60 python tools/quick_gemm.py 2048 9 >> gpurun_out/exp18.log 2>&1 || echo "FAIL $cfg" >> gpurun_out/exp18.log
done
