"""GPU time per tiny ozimmu_dgemm call under env variants (development tool)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2306_11975_b200 as oz  # noqa: E402

h = oz.Handle(0)
out = {"env": os.environ.get("TAG", "")}
for (m, n, k) in [(64, 64, 64), (1024, 1024, 1024)]:
    A = torch.randn(m * k, dtype=torch.float64, device="cuda")
    B = torch.randn(k * n, dtype=torch.float64, device="cuda")
    C = torch.empty(m * n, dtype=torch.float64, device="cuda")
    for _ in range(20):
        h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, 9)
    torch.cuda.synchronize()
    h.timing_enable(64)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, 9)
    e1.record()
    torch.cuda.synchronize()
    ph = h.timing_read(50)
    h.timing_enable(0)
    out[f"{m}_call_us"] = round(e0.elapsed_time(e1) / 50 * 1e3, 1)
    out[f"{m}_gemm_us"] = round(sum(p["gemm_ms"] for p in ph) / len(ph) * 1e3, 1)
    out[f"{m}_slice_us"] = round(sum(p["slice_a_ms"] + p["slice_b_ms"] for p in ph) / len(ph) * 1e3, 1)
print(json.dumps(out), flush=True)
