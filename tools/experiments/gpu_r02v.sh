for sz in 1024 2048 4096; do OZIMMU_STATS=1 python tools/shape_stats.py $sz $sz $sz 9 20 2>&1 | tail -2 | cut -c1-400; done
