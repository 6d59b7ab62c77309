"""DGEMM throughput where the INT32 budget forces K chunks (reading A15): k > 2^14
at s = 9 (development tool).  One JSON line per shape."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_11975_b200 as oz  # noqa: E402

h = oz.Handle(0)
for (m, n, k, s) in [(8192, 8192, 32768, 9), (8192, 8192, 32768, 8), (4096, 4096, 131072, 9),
                     (8192, 8192, 16384, 9)]:
    g = torch.Generator(device="cuda").manual_seed(k)
    A = torch.rand(m * k, dtype=torch.float64, device="cuda", generator=g) - 0.5
    B = torch.rand(k * n, dtype=torch.float64, device="cuda", generator=g) - 0.5
    C = torch.empty(m * n, dtype=torch.float64, device="cuda")
    h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    r = h.report()
    print(json.dumps({"m": m, "n": n, "k": k, "s": s, "tflops": round(2.0 * m * n * k / ms / 1e9, 2),
                      "ms": round(ms, 2), "k_chunks": r["k_chunks"], "acc_regions": r["acc_regions"],
                      "tile_n": r["tile_n"]}), flush=True)
