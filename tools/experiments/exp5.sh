for cfg in "16384 9" "8192 9" "16384 13" "16384 7" "4096 9"; do
timeout 600 python tools/ab.py $cfg default default@OZIMMU_CLUSTER=1 --rounds 2 >> gpurun_out/exp5_ab.log 2>&1
done
