timeout 900 python -m pytest tests/test_gpu_split_fused.py tests/test_gpu_parity.py tests/test_gpu_zgemm.py tests/test_gpu_fuzz.py tests/test_gpu_bigk.py tests/test_gpu_streamk.py -q -x 2>&1 | tail -2
for cx in 1 0; do
OZIMMU_EXACT_LEVELS=$cx python tools/shape_stats.py 16384 16384 16384 9 5 | sed "s/^/cx$cx /"
OZIMMU_EXACT_LEVELS=$cx python tools/shape_stats.py 1048576 512 512 8 10 | sed "s/^/cx$cx /"
OZIMMU_EXACT_LEVELS=$cx python tools/shape_stats.py 1024 1024 1024 9 50 | sed "s/^/cx$cx /"
OZIMMU_EXACT_LEVELS=$cx python tools/shape_stats.py 2048 2048 2048 9 30 | sed "s/^/cx$cx /"
done
