"""PCIe copy rates the host pipeline depends on (development tool): contiguous H2D/D2H from
pinned memory and the 2-D strided row-block copy ozimmu_dgemm_host uses for op(A) rows."""
import json
import torch

N = 16384
h = torch.empty(N * N, dtype=torch.float64).pin_memory()
d = torch.empty(N * N, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def t(fn, nbytes, reps=3):
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9


out = {}
out["h2d_contig_GBs"] = t(lambda: d.copy_(h, non_blocking=True), 8 * N * N)
out["d2h_contig_GBs"] = t(lambda: h.copy_(d, non_blocking=True), 8 * N * N)
# row block of a column-major m x k matrix: 1024 rows of every column (8 KB segments)
hv = h.view(N, N)  # hv[col, row] in column-major terms
dv = d.view(N, N)
rb = 1024
import ctypes as ct
import os
import nvidia.cuda_runtime as _cr
rt = ct.CDLL(os.path.join(os.path.dirname(_cr.__file__), "lib", "libcudart.so.12"))
rt.cudaMemcpy2DAsync.argtypes = [ct.c_void_p, ct.c_size_t, ct.c_void_p, ct.c_size_t, ct.c_size_t,
                                 ct.c_size_t, ct.c_int, ct.c_void_p]
stream = torch.cuda.current_stream().cuda_stream


def copy2d(rows):  # cudaMemcpy2DAsync of `rows` rows of every column (column-major, ld N)
    rc = rt.cudaMemcpy2DAsync(d.data_ptr(), 8 * rows, h.data_ptr(), 8 * N, 8 * rows, N, 1, stream)
    assert rc == 0, rc


for rb in (512, 1024, 2048):
    out[f"h2d_rowblock_memcpy2d_{rb}rows_GBs"] = t(lambda: copy2d(rb), 8 * N * rb, reps=8)
s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    with torch.cuda.stream(s0):
        d[: N * N // 2].copy_(h[: N * N // 2], non_blocking=True)
    with torch.cuda.stream(s1):
        h[N * N // 2:].copy_(d[N * N // 2:], non_blocking=True)
    torch.cuda.synchronize()


out["bidir_total_GBs"] = t(both, 8 * N * N)
print(json.dumps(out))
