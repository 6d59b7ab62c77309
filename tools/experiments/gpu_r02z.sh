timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_zgemm.py tests/test_gpu_fuzz.py tests/test_gpu_bigk.py tests/test_gpu_batched.py -q -x 2>&1 | tail -2
V=paper_2306_11975_b200/variants/libozimmu_nopipe.so
for rep in 1 2; do
for lib in "" $V; do
  OZIMMU_LIB=$lib python tools/shape_stats.py 16384 16384 16384 9 5 | sed "s|^|[$lib] |" | cut -c1-160
  OZIMMU_LIB=$lib python tools/shape_stats.py 1024 1024 1024 9 100 | sed "s|^|[$lib] |" | cut -c1-160
  OZIMMU_LIB=$lib python tools/shape_stats.py 2048 2048 2048 9 50 | sed "s|^|[$lib] |" | cut -c1-160
done; done
