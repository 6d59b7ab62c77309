import os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2306_11975_b200 as oz
N = int(sys.argv[1]); s = int(sys.argv[2])
h = oz.Handle(0)
A = torch.randn(N, N, dtype=torch.float64, device="cuda")
B = torch.randn(N, N, dtype=torch.float64, device="cuda")
C = torch.empty(N, N, dtype=torch.float64, device="cuda")
h.dgemm("N", "N", N, N, N, 1.0, A, N, B, N, 0.0, C, N, s)
torch.cuda.synchronize()
print("ok", os.environ.get("OZIMMU_B_STAGES"), os.environ.get("OZIMMU_A_STAGES"), os.environ.get("OZIMMU_CLUSTER"), float(C.abs().sum()))
