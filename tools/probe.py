"""Quick throughput probe: ozimmu_dgemm vs cuBLAS DGEMM (CUDA events)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2306_11975_b200 as oz

def t_ms(fn, warm=2, it=5):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(it):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort(); return ts[len(ts)//2]

h = oz.Handle(0)
sizes = [int(x) for x in (sys.argv[1:] or ["4096", "8192", "16384"])]
for N in sizes:
    A = torch.randn(N, N, dtype=torch.float64, device="cuda")
    B = torch.randn(N, N, dtype=torch.float64, device="cuda")
    C = torch.empty(N, N, dtype=torch.float64, device="cuda")
    fl = 2.0 * N ** 3
    res = {"N": N}
    for s in (7, 9, 13):
        ms = t_ms(lambda: h.dgemm("N", "N", N, N, N, 1.0, A, N, B, N, 0.0, C, N, s))
        res[f"oz_s{s}_tflops"] = round(fl / ms / 1e9, 2)
        res[f"oz_s{s}_ms"] = round(ms, 3)
        res[f"s{s}_report"] = h.report()
    ms = t_ms(lambda: torch.matmul(A, B, out=C))
    res["cublas_dgemm_tflops"] = round(fl / ms / 1e9, 2)
    print(json.dumps(res), flush=True)
