timeout 900 python -m pytest tests/test_gpu_split_fused.py tests/test_gpu_parity.py tests/test_gpu_zgemm.py tests/test_gpu_auto.py tests/test_gpu_auto_acc.py tests/test_gpu_batched.py -q -x 2>&1 | tail -2
SZ=16384 IT=4 python tools/auto_step_probe.py
python tools/split_bench.py --sizes 16384,8192,2048
