"""One DGEMM shape, device-timed, with the per-phase split (and the kernel's stall counters
when OZIMMU_STATS=1).  usage: python tools/shape_stats.py m n k s [iters]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_11975_b200 as oz  # noqa: E402

m, n, k, s = (int(x) for x in sys.argv[1:5])
it = int(sys.argv[5]) if len(sys.argv) > 5 else 10
h = oz.Handle(0)
h.set_stream(torch.cuda.current_stream())
A = torch.rand(m * k, dtype=torch.float64, device="cuda") - 0.5
B = torch.rand(k * n, dtype=torch.float64, device="cuda") - 0.5
C = torch.empty(m * n, dtype=torch.float64, device="cuda")
call = lambda: h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, s)  # noqa: E731
for _ in range(2):
    call()
torch.cuda.synchronize()
h.timing_enable(it)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(it):
    call()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / it
ph = h.timing_read(it)
h.timing_enable(0)
rep = h.report()
print(json.dumps({"m": m, "n": n, "k": k, "s": s, "tflops": round(2.0 * m * n * k / ms / 1e9, 2),
                  "ms": round(ms, 4), "gemm_ms": round(sum(p["gemm_ms"] for p in ph) / len(ph), 4),
                  "slice_ms": round(sum(max(p["slice_a_ms"], p["slice_b_ms"]) for p in ph) / len(ph), 4),
                  "tile_n": rep["tile_n"], "env": {k2: v for k2, v in os.environ.items()
                                                    if k2.startswith("OZIMMU")}}), flush=True)
