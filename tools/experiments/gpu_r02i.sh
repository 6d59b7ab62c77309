for gm in 8 16 32 74 148; do
OZIMMU_GROUP_M=$gm python tools/shape_stats.py 1048576 512 512 8 10 2>&1 | tail -1
done
for gm in 8 32 148; do
OZIMMU_GROUP_M=$gm C5_DS=8 C5_SS=8 C5_IT=3 python tools/c5_sweep.py 2>&1 | tail -1 | sed "s/^/gm$gm /"
done
