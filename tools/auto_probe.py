"""One INT8-AUTO (accuracy rule) call on the C4 workload, for an ncu launch list of the
statistics kernels (development tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_11975_b200 as oz  # noqa: E402
import synth  # noqa: E402

m = n = k = int(os.environ.get("SZ", "16384"))
A = torch.from_numpy(synth.gen_phi(m, k, 0.5, 401).ravel(order="F")).cuda()
B = torch.from_numpy(synth.gen_phi(k, n, 0.5, 402).ravel(order="F")).cuda()
h = oz.Handle(0)
rule = os.environ.get("RULE", "acc")
if rule == "loss":
    h.set_auto(0.0, 18)
else:
    h.set_auto_accuracy(1.0, 18)
for _ in range(2):
    s = h.auto_splits("N", "N", m, n, k, A, m, B, k)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    s = h.auto_splits("N", "N", m, n, k, A, m, B, k)
e1.record()
torch.cuda.synchronize()
print({"rule": rule, "s": s, "auto_splits_ms": e0.elapsed_time(e1) / 3}, flush=True)
