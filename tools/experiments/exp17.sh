timeout 900 python tools/ab.py 16384 9 default default@OZIMMU_B_STAGES=3 --rounds 2 > gpurun_out/exp17_ab.log 2>&1
OZIMMU_STATS=1 OZIMMU_B_STAGES=3 timeout 200 python tools/stats_run.py 16384 9 > gpurun_out/exp17_stats.log 2>&1
