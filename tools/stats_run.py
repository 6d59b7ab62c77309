import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2306_11975_b200 as oz
N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
s = int(sys.argv[2]) if len(sys.argv) > 2 else 9
h = oz.Handle(0)
A = torch.randn(N, N, dtype=torch.float64, device="cuda")
B = torch.randn(N, N, dtype=torch.float64, device="cuda")
C = torch.empty(N, N, dtype=torch.float64, device="cuda")
for _ in range(3):
    h.dgemm("N", "N", N, N, N, 1.0, A, N, B, N, 0.0, C, N, s)
torch.cuda.synchronize()
