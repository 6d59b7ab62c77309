timeout 600 python -m pytest tests/test_gpu_host.py -x -q > gpurun_out/exp39_tests.log 2>&1
for g in 1 0 1 0; do
OZIMMU_HOST_GROW=$g timeout 300 python - >> gpurun_out/exp39_host.log 2>&1 <<'PY'
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2306_11975_b200 as oz
N = 16384
rng = np.random.default_rng(1)
A = torch.from_numpy(rng.standard_normal((N, N))).pin_memory()
B = torch.from_numpy(rng.standard_normal((N, N))).pin_memory()
C = torch.empty((N, N), dtype=torch.float64).pin_memory()
h = oz.Handle(0)
f = lambda: h.dgemm_host("N", "N", N, N, N, 1.0, A, N, B, N, 0.0, C, N, 9)
f(); f()
ts = []
for _ in range(5):
    t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
ts.sort()
print(json.dumps({"grow": os.environ["OZIMMU_HOST_GROW"], "ms": ts[2] * 1e3, "tflops": 2 * N**3 / ts[2] / 1e12}))
PY
done
