"""INT8-AUTO call cost at C4 (development probe): back-to-back ozimmu_dgemm calls with s = 9
fixed and with num_slices = 0 (accuracy rule), device-timed, with the library's phase marks,
plus ozimmu_auto_splits alone."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_11975_b200 as oz  # noqa: E402
import synth  # noqa: E402

n = int(os.environ.get("SZ", "16384"))
it = int(os.environ.get("IT", "6"))
A = torch.from_numpy(synth.gen_phi(n, n, 0.5, 401).ravel(order="F")).cuda()
B = torch.from_numpy(synth.gen_phi(n, n, 0.5, 402).ravel(order="F")).cuda()
C = torch.empty(n * n, dtype=torch.float64, device="cuda")
h = oz.Handle(0)
h.set_stream(torch.cuda.current_stream())
h.set_auto_accuracy(1.0, 18)
for s in (9, 0, 9, 0):
    call = lambda: h.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, s)  # noqa: E731
    call()
    torch.cuda.synchronize()
    h.timing_enable(it)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(it):
        call()
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / it * 1e3
    ph = h.timing_read(it)
    h.timing_enable(0)
    print(json.dumps({"s": s, "chosen": h.report()["num_slices"], "ms": e0.elapsed_time(e1) / it,
                      "wall_ms": wall,
                      "gemm_ms": sum(p["gemm_ms"] for p in ph) / len(ph),
                      "slice_ms": sum(max(p["slice_a_ms"], p["slice_b_ms"]) for p in ph) / len(ph)}),
          flush=True)
t0 = time.perf_counter()
for _ in range(it):
    h.auto_splits("N", "N", n, n, n, A, n, B, n)
print(json.dumps({"auto_splits_wall_ms": (time.perf_counter() - t0) / it * 1e3}))
