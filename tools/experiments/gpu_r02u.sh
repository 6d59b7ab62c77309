timeout 900 python -m pytest tests/test_gpu_split_fused.py tests/test_gpu_parity.py tests/test_gpu_zgemm.py tests/test_gpu_fuzz.py tests/test_gpu_bigk.py -q -x 2>&1 | tail -2
python tools/split_bench.py --sizes 16384 --s 12
C5_DS=8,12 C5_SS=12 C5_IT=3 python tools/c5_sweep.py | cut -c1-330
