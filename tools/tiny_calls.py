import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2306_11975_b200 as oz
h = oz.Handle(0)
for (m, n, k) in [(64, 64, 64), (1024, 1024, 1024)]:
    A = torch.randn(m * k, dtype=torch.float64, device="cuda")
    B = torch.randn(k * n, dtype=torch.float64, device="cuda")
    C = torch.empty(m * n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        h.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, 9)
torch.cuda.synchronize()
