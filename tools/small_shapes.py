"""Effective TFLOP/s of ozimmu_dgemm at the small end of the paper's target range (P:367-368,
2^11 <= m, n, k; P:621-622 flags m <= 2^11 under-utilisation), with cuBLAS DGEMM beside it
(development tool; --quick: fewer iterations for ncu launch lists).  One JSON line per shape."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_11975_b200 as oz  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true")
ap.add_argument("--s", type=int, default=9)
ap.add_argument("--shapes", default="1024,1536,2048,3072,4096")
ap.add_argument("--warm-s", type=float, default=0.0,
                help="seconds of back-to-back calls before timing each shape (clock ramp-up)")
args = ap.parse_args()
it = 3 if args.quick else 30


def t_ms(fn, n_it):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n_it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n_it


h = oz.Handle(0)
h.set_stream(torch.cuda.current_stream())
for sz in [int(x) for x in args.shapes.split(",")]:
    m = n = k = sz
    g = torch.Generator(device="cuda").manual_seed(sz)
    A = torch.rand(m * k, dtype=torch.float64, device="cuda", generator=g) - 0.5
    B = torch.rand(k * n, dtype=torch.float64, device="cuda", generator=g) - 0.5
    C = torch.empty(m * n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, args.s)
    torch.cuda.synchronize()
    if args.warm_s > 0:
        import time
        t_end = time.perf_counter() + args.warm_s
        while time.perf_counter() < t_end:
            for _ in range(20):
                h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, args.s)
            torch.cuda.synchronize()
    # the call time WITHOUT the phase events (recording 5 events per call costs ~15 us at
    # 1024^3); the phase split from a second loop with timing on
    ms = t_ms(lambda: h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, args.s), it)
    h.timing_enable(it + 1)
    t_ms(lambda: h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, args.s), it)
    ph = h.timing_read(it + 1)
    h.timing_enable(0)
    rep = h.report()
    Am, Bm = A.view(k, m).t(), B.view(n, k).t()
    cms = t_ms(lambda: torch.matmul(Am, Bm), it)
    fl = 2.0 * m * n * k
    print(json.dumps({
        "m": m, "n": n, "k": k, "s": args.s, "ozimmu_tflops": round(fl / ms / 1e9, 2),
        "cublas_tflops": round(fl / cms / 1e9, 2), "ozimmu_us": round(ms * 1e3, 1),
        "slice_us": round(sum(max(p["slice_a_ms"], p["slice_b_ms"]) for p in ph) / len(ph) * 1e3, 1),
        "gemm_us": round(sum(p["gemm_ms"] for p in ph) / len(ph) * 1e3, 1),
        "tile_n": rep["tile_n"], "launches": rep["launches"]}), flush=True)
