"""Child process for tests/test_gpu_streamk.py: run a set of Ozaki GEMMs with the stream-K
schedule forced on or off (OZIMMU_SK is read once per process) and save the results."""
import sys

import numpy as np
import torch

sys.path.insert(0, sys.argv[2])
import paper_2306_11975_b200 as oz  # noqa: E402
import synth  # noqa: E402

CASES = [  # (ta, tb, m, n, k, s, phi)
    ("N", "N", 200, 333, 1000, 9, 1.0),
    ("T", "N", 300, 500, 700, 13, 0.5),
    ("N", "T", 1000, 990, 1024, 9, 0.5),
    ("T", "T", 129, 49, 33, 8, 1.0),
    ("N", "N", 130, 96, 16384, 9, 0.5),     # two INT32 regions per level (T = 2)
    ("N", "N", 1, 300, 4097, 11, 2.0),
    ("N", "N", 2048, 2048, 2048, 9, 0.5),
]


def main(out):
    h = oz.Handle(0)
    res = {}
    for i, (ta, tb, m, n, k, s, phi) in enumerate(CASES):
        A = synth.gen_phi(*((m, k) if ta == "N" else (k, m)), phi, 900 + i)
        B = synth.gen_phi(*((k, n) if tb == "N" else (n, k)), phi, 950 + i)
        Cin = synth.gen_phi(m, n, 0.5, 990 + i)
        dA = torch.from_numpy(A.ravel(order="F").copy()).cuda()
        dB = torch.from_numpy(B.ravel(order="F").copy()).cuda()
        dC = torch.from_numpy(Cin.ravel(order="F").copy()).cuda()
        h.dgemm(ta, tb, m, n, k, 1.5, dA, A.shape[0], dB, B.shape[0], -0.5, dC, m, s)
        torch.cuda.synchronize()
        res[f"C{i}"] = dC.cpu().numpy().reshape(n, m).T
        if i < 3:  # exact level sums through the same schedule
            L = torch.empty(s * m * n, dtype=torch.int64, device="cuda")
            h.debug_level_sums(ta, tb, m, n, k, dA, A.shape[0], dB, B.shape[0], s, L)
            torch.cuda.synchronize()
            res[f"L{i}"] = L.cpu().numpy().reshape(s, n, m).transpose(0, 2, 1)
    # ZGEMM through the same kernel (EPI_ZGEMM)
    Az = synth.gen_phi_complex(300, 200, 0.5, 7)
    Bz = synth.gen_phi_complex(200, 170, 0.5, 8)
    zA = torch.from_numpy(Az.ravel(order="F").copy()).cuda()
    zB = torch.from_numpy(Bz.ravel(order="F").copy()).cuda()
    zC = torch.zeros(300 * 170, dtype=torch.complex128, device="cuda")
    h.zgemm("N", "N", 300, 170, 200, 1.0, zA, 300, zB, 200, 0.0, zC, 300, 9)
    torch.cuda.synchronize()
    res["Z"] = zC.cpu().numpy().reshape(170, 300).T
    np.savez(out, **res)
    h.close()


if __name__ == "__main__":
    main(sys.argv[1])
