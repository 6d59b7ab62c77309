timeout 900 python tools/ab.py 16384 9 default default@OZIMMU_KSYNC=32 default@OZIMMU_KSYNC=8 --rounds 2 > gpurun_out/exp32_ab.log 2>&1
