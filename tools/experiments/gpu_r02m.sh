nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 100 > gpurun_out/r02m_clocks.txt &
SMI=$!
python tools/small_shapes.py --shapes 1024,2048 | sed "s/^/cold /"
python tools/small_shapes.py --shapes 1024,2048 --warm-s 1.0 | sed "s/^/warm /"
OZIMMU_STATS=1 python tools/shape_stats.py 1024 1024 1024 9 3 2>&1 | tail -2
kill $SMI
sort gpurun_out/r02m_clocks.txt | uniq -c | sort -rn | head -8
OZIMMU_CLUSTER_N=4 C5_DS=8 C5_SS=8 C5_IT=3 python tools/c5_sweep.py | sed "s/^/cln4 /"
OZIMMU_CLUSTER_N=4 python tools/shape_stats.py 1048576 512 512 8 10 | sed "s/^/cln4 /"
