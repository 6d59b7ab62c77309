import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2306_11975_b200 as oz
import synth
N = 16384
A = torch.from_numpy(synth.gen_phi(N, N, 0.5, 401).ravel(order="F")).pin_memory()
B = torch.from_numpy(synth.gen_phi(N, N, 0.5, 402).ravel(order="F")).pin_memory()
C = torch.empty(N * N, dtype=torch.float64).pin_memory()
h = oz.Handle(0)
h.set_auto(1.0, 20)
f = lambda: h.dgemm_host("N", "N", N, N, N, 1.0, A, N, B, N, 0.0, C, N, 0)
f(); f()
ts = []
for _ in range(4):
    t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
ts.sort()
print(json.dumps({"auto_T1_host_ms": ts[1] * 1e3, "tflops": 2 * N**3 / ts[1] / 1e12, "s": h.report()["num_slices"]}))
