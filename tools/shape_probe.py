"""Effective TFLOP/s of ozimmu_dgemm over shapes (development tool): m = n = 16384 with small
k (the tile-switch / epilogue share grows as k shrinks), and cuBLAS DGEMM beside it."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2306_11975_b200 as oz  # noqa: E402


def t_ms(fn, it=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


h = oz.Handle(0)
shapes = [(16384, 16384, 1024), (16384, 16384, 2048), (16384, 16384, 4096), (4096, 4096, 4096),
          (2048, 2048, 2048), (1024, 1024, 1024)]
for m, n, k in shapes:
    A = torch.randn(m * k, dtype=torch.float64, device="cuda")
    B = torch.randn(k * n, dtype=torch.float64, device="cuda")
    C = torch.empty(m * n, dtype=torch.float64, device="cuda")
    ms = t_ms(lambda: h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, 9))
    Am, Bm = A.view(k, m).t(), B.view(n, k).t()
    cms = t_ms(lambda: torch.matmul(Am, Bm))
    fl = 2.0 * m * n * k
    print(json.dumps({"m": m, "n": n, "k": k, "ozimmu_tflops": round(fl / ms / 1e9, 2),
                      "cublas_tflops": round(fl / cms / 1e9, 2), "ozimmu_ms": round(ms, 3)}),
          flush=True)

# per-call overhead: a tiny call (GPU work negligible), host wall time per call
import time  # noqa: E402
m = n = k = 64
A = torch.randn(m * k, dtype=torch.float64, device="cuda")
B = torch.randn(k * n, dtype=torch.float64, device="cuda")
C = torch.empty(m * n, dtype=torch.float64, device="cuda")
for _ in range(10):
    h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, 9)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, 9)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
gms = t_ms(lambda: h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, 9), it=200)
print(json.dumps({"tiny_call_host_us": round((t1 - t0) / 200 * 1e6, 1),
                  "tiny_call_total_us": round((t2 - t0) / 200 * 1e6, 1),
                  "tiny_call_gpu_event_us": round(gms * 1e3, 1)}), flush=True)
