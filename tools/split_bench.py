"""Slicing kernels alone (A2 + A3): ozimmu_slice_b on a k x n operand, contiguous vectors
(transB = N) and strided vectors (transB = T), device-timed with CUDA events; algorithmic
HBM bytes = (8 + s) per element + 4 per vector.  One JSON line per (layout, size).
usage: python tools/split_bench.py [--sizes 16384,8192] [--s 9]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_11975_b200 as oz  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="16384,8192,2048,1024")
ap.add_argument("--s", type=int, default=9)
ap.add_argument("--it", type=int, default=20)
args = ap.parse_args()

h = oz.Handle(0)
h.set_stream(torch.cuda.current_stream())
for sz in [int(x) for x in args.sizes.split(",")]:
    k = n = sz
    B = torch.rand(k * n, dtype=torch.float64, device="cuda") - 0.5
    buf = torch.empty(oz.b_slices_bytes(n, k, args.s), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for tb in ["N", "T"]:
        for _ in range(3):
            h.slice_b(tb, k, n, B, k if tb == "N" else n, args.s, buf)
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.it):
            flush.zero_()  # L2 flush between timed calls
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            h.slice_b(tb, k, n, B, k if tb == "N" else n, args.s, buf)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        ms = ts[len(ts) // 2]
        byts = (8 + args.s) * k * n + 4 * n
        print(json.dumps({"layout": "contiguous" if tb == "N" else "strided", "k": k, "n": n,
                          "s": args.s, "ms_median": round(ms, 4), "ms_min": round(ts[0], 4),
                          "GBps": round(byts / ms / 1e6, 1),
                          "fused": os.environ.get("OZIMMU_SPLIT_FUSED", "1"),
                          "launches": h.report()["launches"]}), flush=True)
