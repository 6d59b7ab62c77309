timeout 900 python -m pytest tests/test_gpu_zgemm.py tests/test_gpu_batched.py tests/test_gpu_fuzz.py tests/test_gpu_split_fused.py -q -x 2>&1 | tail -2
C5_DS=8,10,12 C5_SS=8,12 C5_IT=3 python tools/c5_sweep.py | cut -c1-330
