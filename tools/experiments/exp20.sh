for N in 2560 3072 4096 6144; do
  OZIMMU_A_STAGES=3 timeout 60 python tools/quick_gemm.py $N 9 >> gpurun_out/exp20.log 2>&1 && echo "PASS N=$N" >> gpurun_out/exp20.log || echo "FAIL N=$N" >> gpurun_out/exp20.log
done
OZIMMU_A_STAGES=3 timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/quick_gemm.py 4096 9 > gpurun_out/exp20_san.log 2>&1
echo "san rc=$?" >> gpurun_out/exp20_san.log
