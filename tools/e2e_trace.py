"""Timeline of one host-buffer call (ozimmu_dgemm_host) at C4 size: OZIMMU_HOST_TRACE=1 makes
the library print when each A row block / B column chunk landed and when each C region's GEMM
ran and came back (ms from the call's start).  Development probe."""
import os
import sys
import time

os.environ.setdefault("OZIMMU_HOST_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_11975_b200 as oz  # noqa: E402

n = int(os.environ.get("SZ", "16384"))
s = int(os.environ.get("S", "9"))
A = (torch.rand(n * n, dtype=torch.float64) - 0.5).pin_memory()
B = (torch.rand(n * n, dtype=torch.float64) - 0.5).pin_memory()
C = torch.empty(n * n, dtype=torch.float64).pin_memory()
h = oz.Handle(0)
for i in range(3):
    t0 = time.perf_counter()
    h.dgemm_host("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, s)
    dt = time.perf_counter() - t0
    print(f"call {i}: {dt * 1e3:.1f} ms = {2.0 * n ** 3 / dt / 1e12:.1f} TFLOP/s", file=sys.stderr,
          flush=True)
