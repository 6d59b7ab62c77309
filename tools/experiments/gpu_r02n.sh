for cv in -1 100 0; do
OZIMMU_SPLIT_CARVEOUT=$cv python tools/small_shapes.py --shapes 1024,2048 | sed "s/^/cv$cv /"
done
OZIMMU_NO_WAVE_SYNC=1 OZIMMU_SPLIT_CARVEOUT=100 python tools/small_shapes.py --shapes 1024,2048 | sed "s/^/cv100nows /"
