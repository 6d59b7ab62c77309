"""NEXT row f4 on the GPU: A * A_dag -- Ozaki (tcgen05 path) is more accurate
than cuBLAS DGEMM against the double-double reference, and bit-exact vs the oracle."""
import numpy as np
import pytest

import oracle as O
import synth
from gpu_util import dev, host

pytestmark = pytest.mark.gpu


def test_invpair_gpu_beats_cublas():
    import torch
    import paper_2306_11975_b200 as oz
    h = oz.Handle(0)
    n = 512
    A, Ad = synth.gen_inverse_pair(n, 3)
    rows = np.arange(0, n, 8)
    hi, lo = O.dd_gemm("N", "N", n, n, n, A, n, Ad, n, rows=rows)
    cub = (torch.from_numpy(A).cuda() @ torch.from_numpy(Ad).cuda()).cpu().numpy()
    st_cub = O.err_stats(cub[rows], hi, lo)
    res = {}
    for s in (9, 11, 13):
        dC = torch.zeros(n * n, dtype=torch.float64, device="cuda")
        h.dgemm("N", "N", n, n, n, 1.0, dev(A), n, dev(Ad), n, 0.0, dC, n, s)
        torch.cuda.synchronize()
        C = host(dC, n, n)
        res[s] = O.err_stats(C[rows], hi, lo)
        if s == 11:
            ref = O.dgemm("N", "N", n, n, n, 1.0, A, n, Ad, n, 0.0, np.zeros((n, n), order="F"),
                          n, s, rows=rows[:16])
            assert np.array_equal(C[rows[:16]], ref[rows[:16]])
    assert res[11]["mean_rel"] < st_cub["mean_rel"], (res, st_cub)
    assert res[13]["mean_rel"] < st_cub["mean_rel"]
