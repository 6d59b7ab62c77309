"""Child process for tests/test_gpu_sanitizer.py: a few small Ozaki GEMMs through the C ABI
(ragged tiles, both MMA issuers, CTA pairs, the stream-K fixup, the K-chunked INT32 budget
path and the double-buffered TMEM accumulators), run under compute-sanitizer.  Prints OK
after checking every result against the oracle
(the run also checks that the instrumented kernels still compute the right bits)."""
import sys

import numpy as np
import torch

sys.path.insert(0, sys.argv[1])
import oracle as O  # noqa: E402
import paper_2306_11975_b200 as oz  # noqa: E402
import synth  # noqa: E402

CASES = [("N", "N", 256, 192, 512, 9), ("T", "N", 130, 100, 300, 13),
         ("N", "T", 64, 400, 200, 7), ("N", "N", 40, 24, 140000, 7),
         # two TMEM accumulator buffers alternating over several tiles per CTA (short K)
         ("T", "N", 1500, 640, 256, 4)]

h = oz.Handle(0)
for i, (ta, tb, m, n, k, s) in enumerate(CASES):
    A = synth.gen_phi(*((m, k) if ta == "N" else (k, m)), 1.0, 40 + i)
    B = synth.gen_phi(*((k, n) if tb == "N" else (n, k)), 1.0, 50 + i)
    Cin = synth.gen_phi(m, n, 1.0, 60 + i)
    dA = torch.from_numpy(A.ravel(order="F").copy()).cuda()
    dB = torch.from_numpy(B.ravel(order="F").copy()).cuda()
    dC = torch.from_numpy(Cin.ravel(order="F").copy()).cuda()
    h.dgemm(ta, tb, m, n, k, 1.25, dA, A.shape[0], dB, B.shape[0], 0.5, dC, m, s)
    torch.cuda.synchronize()
    got = dC.cpu().numpy().reshape(n, m).T
    rows = None if m * n * k < 10 ** 8 else [0, m - 1]
    ref = O.dgemm(ta, tb, m, n, k, 1.25, A, A.shape[0], B, B.shape[0], 0.5, Cin, m, s, rows=rows)
    sel = slice(None) if rows is None else rows
    assert np.array_equal(got[sel], ref[sel]), (i, ta, tb, m, n, k, s)
h.close()
print("OK", flush=True)
