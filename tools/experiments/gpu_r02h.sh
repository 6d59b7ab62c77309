mkdir -p gpurun_out
for acc in 0 1; do
OZIMMU_ACC2=$acc OZIMMU_STATS=1 python tools/shape_stats.py 1048576 512 512 8 3 2>&1 | tail -2
OZIMMU_ACC2=$acc python tools/shape_stats.py 1048576 512 512 8 10 2>&1 | tail -1
done
OZIMMU_STATS=1 python tools/shape_stats.py 16384 16384 16384 9 1 2>&1 | tail -2
