"""Small problems with and without CUDA-graph replay (development tool): the per-call time of
ozimmu_dgemm issued eagerly, and of the same calls captured once into a CUDA graph (10 calls
per graph) and replayed -- the difference is the host launch / stream-ordering overhead that a
caller can remove by capturing (a fixed-s call makes no host synchronisation).
One JSON line per shape.  usage: python tools/graph_small.py [--shapes 1024,2048] [--s 9]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_11975_b200 as oz  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="1024,1536,2048,4096")
ap.add_argument("--s", type=int, default=9)
ap.add_argument("--per-graph", type=int, default=10)
ap.add_argument("--replays", type=int, default=20)
args = ap.parse_args()


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


side = torch.cuda.Stream()
h = oz.Handle(0)
h.set_stream(side)
for sz in [int(x) for x in args.shapes.split(",")]:
    m = n = k = sz
    g = torch.Generator(device="cuda").manual_seed(sz)
    A = torch.rand(m * k, dtype=torch.float64, device="cuda", generator=g) - 0.5
    B = torch.rand(k * n, dtype=torch.float64, device="cuda", generator=g) - 0.5
    C = torch.empty(m * n, dtype=torch.float64, device="cuda")

    def call():
        h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, args.s)

    with torch.cuda.stream(side):
        for _ in range(3):
            call()  # sizes the workspace before capture
        torch.cuda.synchronize()
        eager_ms = timed(call, 30)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            for _ in range(args.per_graph):
                call()
        graph_ms = timed(graph.replay, args.replays) / args.per_graph
    fl = 2.0 * m * n * k
    print(json.dumps({"m": m, "n": n, "k": k, "s": args.s,
                      "eager_us": round(eager_ms * 1e3, 1), "graph_us": round(graph_ms * 1e3, 1),
                      "eager_tflops": round(fl / eager_ms / 1e9, 2),
                      "graph_tflops": round(fl / graph_ms / 1e9, 2)}), flush=True)
h.close()
