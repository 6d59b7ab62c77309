"""Child process for tests/test_gpu_split_fused.py: slicing (debug_split), DGEMM and ZGEMM
cases run under the knobs of the environment (OZIMMU_SPLIT_FUSED, OZIMMU_SPLIT_PANEL_KB,
OZIMMU_ACC2 are read once per process); results saved for the parent."""
import sys

import numpy as np
import torch

sys.path.insert(0, sys.argv[2])
import paper_2306_11975_b200 as oz  # noqa: E402
import synth  # noqa: E402

# debug_split: (op, is_rows, rows, kdim, s); vector r element l = op(M)(r, l) (A) / (l, r) (B)
SPLITS = [("N", 1, 300, 1000, 9), ("T", 1, 300, 3000, 9), ("N", 0, 77, 2100, 13),
          ("T", 0, 100, 700, 7), ("N", 1, 40, 4097, 17), ("N", 1, 1000, 333, 9),
          ("T", 1, 33, 20000, 9), ("N", 0, 5, 4096, 20), ("T", 0, 257, 128, 5),
          # 96-bit fraction window of the fast digit path (10 <= s <= 13 at w = 7)
          ("N", 1, 70, 700, 10), ("T", 1, 45, 2500, 11), ("N", 0, 90, 3000, 12),
          ("T", 0, 64, 300, 13),
          # larger strided operands (rows of op(A) with transA = N, columns of op(B) with T)
          ("N", 1, 1100, 1500, 9), ("T", 0, 700, 3000, 13)]
# dgemm: (ta, tb, m, n, k, s)
DGEMMS = [("N", "N", 300, 200, 5000, 9), ("T", "T", 129, 300, 2500, 13),
          ("N", "T", 64, 70, 20000, 9), ("T", "N", 1, 2049, 2048, 7),
          # short K, s <= 8: two TMEM accumulator buffers (N_c = 32 / default width)
          ("N", "N", 1000, 300, 1000, 8), ("T", "N", 257, 129, 64, 4), ("N", "T", 600, 97, 300, 3),
          # k > 2^17: w = 6 digits
          ("N", "T", 24, 40, 140000, 9),
          # op(A) strided, ~1000 rows
          ("N", "N", 1300, 64, 1200, 9),
          # both operands strided, 1024 < k_pad <= 2048: clusters of 15 CTAs in the small path
          ("N", "T", 200, 150, 1800, 9)]
# zgemm: (ta, tb, m, n, k, s)
ZGEMMS = [("N", "N", 200, 96, 1500, 9), ("C", "T", 70, 45, 1100, 12), ("T", "C", 65, 33, 2100, 8),
          ("N", "T", 3000, 64, 256, 8)]


def split_matrix(shape, seed):
    M = synth.gen_phi(*shape, 2.0, seed)
    M.flat[::97] = 0.0
    M.flat[5::211] = 5e-324
    M.flat[7::1001] *= 1e200
    if M.shape[1] > 3:
        M[:, 3] = 0.0
    return M


def main(out):
    h = oz.Handle(0)
    res = {}
    for i, (op, is_rows, rows, kdim, s) in enumerate(SPLITS):
        if is_rows:
            shape = (rows, kdim) if op == "N" else (kdim, rows)
        else:
            shape = (kdim, rows) if op == "N" else (rows, kdim)
        M = split_matrix(shape, 500 + i)
        planes = torch.empty(s * rows * kdim, dtype=torch.int8, device="cuda")
        exps = torch.empty(rows, dtype=torch.int32, device="cuda")
        dM = torch.from_numpy(M.ravel(order="F").copy()).cuda()
        h.debug_split(op, is_rows, rows, kdim, dM, shape[0], s, planes, exps)
        torch.cuda.synchronize()
        res[f"P{i}"] = planes.cpu().numpy().reshape(s, rows, kdim)
        res[f"E{i}"] = exps.cpu().numpy()
    for i, (ta, tb, m, n, k, s) in enumerate(DGEMMS):
        A = synth.gen_phi(*((m, k) if ta == "N" else (k, m)), 1.0, 600 + i)
        B = synth.gen_phi(*((k, n) if tb == "N" else (n, k)), 1.0, 650 + i)
        Cin = synth.gen_phi(m, n, 0.5, 690 + i)
        dA = torch.from_numpy(A.ravel(order="F").copy()).cuda()
        dB = torch.from_numpy(B.ravel(order="F").copy()).cuda()
        dC = torch.from_numpy(Cin.ravel(order="F").copy()).cuda()
        h.dgemm(ta, tb, m, n, k, 1.5, dA, A.shape[0], dB, B.shape[0], -0.5, dC, m, s)
        torch.cuda.synchronize()
        res[f"D{i}"] = dC.cpu().numpy().reshape(n, m).T
    for i, (ta, tb, m, n, k, s) in enumerate(ZGEMMS):
        A = synth.gen_phi_complex(*((m, k) if ta == "N" else (k, m)), 0.5, 700 + i)
        B = synth.gen_phi_complex(*((k, n) if tb == "N" else (n, k)), 0.5, 750 + i)
        Cin = synth.gen_phi_complex(m, n, 0.5, 790 + i)
        z = lambda a: torch.from_numpy(np.ascontiguousarray(a.ravel(order="F"))).cuda()  # noqa
        dC = z(Cin)
        h.zgemm(ta, tb, m, n, k, 0.75 - 1.25j, z(A), A.shape[0], z(B), B.shape[0], 2.0j, dC, m, s)
        torch.cuda.synchronize()
        res[f"Z{i}"] = dC.cpu().numpy().reshape(n, m).T
    np.savez(out, **res)


if __name__ == "__main__":
    main(sys.argv[1])
