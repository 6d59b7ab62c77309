"""BASELINE config 5 sweep: one d-qubit Haar gate on an N = 28-qubit
state vector, ZGEMM matmul-(2^(N-d), 2^d, 2^d), for d in {8, 10, 12, 14} and the slice
counts the paper's INT8-AUTO chose (T = 0: 12-13, T = 1: 8-9), against cuBLAS ZGEMM
(torch.matmul complex128) on the same data.  Effective rate 8mnk/t.  Also records the s each
INT8-AUTO rule picks on this data (loss rule T = 0 / T = 1, reading A17; accuracy rule,
reading A18).  d = 16 is left out: U (2^32 complex) and its slices (s x 2^34 bytes) exceed the
180 GB of one B200.  One JSON line per (d, s); state and gate are generated on the GPU (torch,
seeded): this is a throughput measurement, the parity tests use synth/ inputs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_11975_b200 as oz  # noqa: E402

NQ = 28
DS = [int(x) for x in os.environ.get("C5_DS", "8,10,12,14").split(",")]
SS = [int(x) for x in os.environ.get("C5_SS", "8,9,12,13").split(",")]
IT = int(os.environ.get("C5_IT", "5"))


def t_ms(fn, it):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


h = oz.Handle(0)
h.set_stream(torch.cuda.current_stream())
for d in DS:
    m, n, k = 2 ** (NQ - d), 2 ** d, 2 ** d
    g = torch.Generator(device="cuda").manual_seed(500 + d)
    # state: complex Gaussian, normalised (a random state vector)
    psi = torch.randn(k * m, dtype=torch.complex128, device="cuda", generator=g)
    psi /= torch.linalg.vector_norm(psi)
    Z = torch.randn(k, k, dtype=torch.complex128, device="cuda", generator=g) / 2 ** 0.5
    Q, R = torch.linalg.qr(Z)
    dg = torch.diagonal(R)
    U = (Q * (dg / dg.abs())).contiguous()  # Haar unitary (row-major)
    del Z, Q, R
    # column-major views for the C ABI: A = psi as m x k (ld m), op(B) = U^T (U row-major is
    # U^T column-major, ld k), C = A U^T (m x n)
    dA = psi
    dB = U.reshape(-1)
    dC = torch.empty(m * n, dtype=torch.complex128, device="cuda")
    picks = {}
    for name, setter in (("loss_T0", lambda: h.set_auto(0.0, 18)),
                         ("loss_T1", lambda: h.set_auto(1.0, 18)),
                         ("acc_tau1", lambda: h.set_auto_accuracy(1.0, 18))):
        setter()
        h.zgemm("N", "N", m, n, k, 1.0, dA, m, dB, k, 0.0, dC, m, 0)
        torch.cuda.synchronize()
        picks[name] = h.report()["num_slices"]
    Am = dA.view(k, m).t()
    Bm = dB.view(k, n)  # U row-major: op(B) = U^T -> torch matmul(A, U^T) = A @ U.T
    Bt = U.t()
    cms = t_ms(lambda: torch.matmul(Am, Bt), IT)
    fl = 8.0 * m * n * k
    for s in SS:
        ms = t_ms(lambda: h.zgemm("N", "N", m, n, k, 1.0, dA, m, dB, k, 0.0, dC, m, s), IT)
        rep = h.report()
        h.timing_enable(2)
        h.zgemm("N", "N", m, n, k, 1.0, dA, m, dB, k, 0.0, dC, m, s)
        torch.cuda.synchronize()
        ph = h.timing_read(2)[-1]
        h.timing_enable(0)
        print(json.dumps({"d": d, "nq": NQ, "m": m, "n": n, "k": k, "s": s,
                          "ozimmu_tflops": round(fl / ms / 1e9, 2), "ozimmu_ms": round(ms, 3),
                          "cublas_zgemm_tflops": round(fl / cms / 1e9, 2),
                          "cublas_ms": round(cms, 3), "speedup": round(cms / ms, 3),
                          "tile_n": rep["tile_n"], "k_chunks": rep["k_chunks"],
                          "acc_regions": rep["acc_regions"],
                          "phases_ms": {kk: round(v, 3) for kk, v in ph.items()},
                          "auto_picks": picks}), flush=True)
    del psi, U, dA, dB, dC, Am, Bm, Bt
    torch.cuda.empty_cache()
