timeout 900 python -m pytest tests/test_gpu_auto_rho.py tests/test_gpu_auto_acc.py tests/test_gpu_auto.py tests/test_gpu_host.py -q -x 2>&1 | tail -2
SZ=16384 IT=4 python tools/auto_step_probe.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_resid python tools/auto_probe.py 2>&1 | grep -E "k_resid|duration" | head -8
