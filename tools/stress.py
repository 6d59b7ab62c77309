"""Race detector for the fused GEMM (development tool): repeat the same call many times and
require identical bits every time, across shapes / slice counts; run it under different
OZIMMU_A_STAGES / OZIMMU_CLUSTER settings to shift the timing."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2306_11975_b200 as oz  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
h = oz.Handle(0)
g = torch.Generator(device="cuda").manual_seed(3)
bad = 0
for (m, n, k, s) in [(4096, 4096, 4096, 9), (8192, 8192, 16384, 9), (3000, 5000, 7000, 13),
                     (6144, 2048, 20000, 7)]:
    A = torch.randn(m * k, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(k * n, dtype=torch.float64, device="cuda", generator=g)
    C = torch.empty(m * n, dtype=torch.float64, device="cuda")
    ref = None
    for r in range(reps):
        h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, s)
        torch.cuda.synchronize()
        hs = hashlib.sha1(C.cpu().numpy().tobytes()).hexdigest()
        if ref is None:
            ref = hs
        elif hs != ref:
            bad += 1
            print(f"MISMATCH m={m} n={n} k={k} s={s} rep={r}", flush=True)
    print(f"m={m} n={n} k={k} s={s}: {reps} reps, hash {ref[:12]}", flush=True)
print("STRESS", "FAIL" if bad else "OK", os.environ.get("OZIMMU_A_STAGES"), os.environ.get("OZIMMU_CLUSTER"))
sys.exit(1 if bad else 0)
