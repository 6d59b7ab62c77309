"""Time the INT8-AUTO mantissa-loss scan (ozimmu_auto_splits) and the slicing phases on the
C4 operands (16384^2, phi = 0.5), all four transposes, with CUDA events.  Development tool;
run under gpurun (optionally under ncu for the per-kernel launch list)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2306_11975_b200 as oz  # noqa: E402
import synth  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    A = torch.from_numpy(synth.gen_phi(n, n, 0.5, 401).ravel(order="F")).cuda()
    B = torch.from_numpy(synth.gen_phi(n, n, 0.5, 402).ravel(order="F")).cuda()
    h = oz.Handle(0)
    h.set_stream(torch.cuda.current_stream())
    out = {}
    for ta, tb in [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")]:
        h.set_auto(0.0, 20)
        s = h.auto_splits(ta, tb, n, n, n, A, n, B, n)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            h.auto_splits(ta, tb, n, n, n, A, n, B, n)
        e1.record()
        torch.cuda.synchronize()
        out[ta + tb] = {"s": s, "auto_ms": e0.elapsed_time(e1) / reps}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
