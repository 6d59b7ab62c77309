timeout 900 python tools/ab.py 16384 9 default default@OZIMMU_PREFETCH_KB=1 default@OZIMMU_PREFETCH_KB=2 --rounds 2 > gpurun_out/exp26_ab.log 2>&1
