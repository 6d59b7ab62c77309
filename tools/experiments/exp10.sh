timeout 900 python tools/ab.py 16384 9 default default@OZIMMU_NO_WAVE_SYNC=1 --rounds 2 > gpurun_out/exp10_ab.log 2>&1
OZIMMU_STATS=1 timeout 200 python tools/stats_run.py 16384 9 > gpurun_out/exp10_stats.log 2>&1
OZIMMU_STATS=1 OZIMMU_NO_WAVE_SYNC=1 timeout 200 python tools/stats_run.py 16384 9 >> gpurun_out/exp10_stats.log 2>&1
