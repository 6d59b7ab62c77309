"""NEXT row f4 on the oracle: the zero-cancellation workload A * A_dag.
"The error of INT8xX is smaller than DGEMM since the Ozaki scheme calculates the
cancellation of the high digit part of the resulting mantissa with higher accuracy"
 -- checked against the double-double reference (not the identity)."""
import numpy as np

import oracle as O
import synth


def test_inverse_pair_generator():
    A, Ad = synth.gen_inverse_pair(64, 1)
    assert np.max(np.abs(A @ Ad - np.eye(64))) < 1e-10  # SPEC S:497 residual check


def test_ozaki_beats_fp64_on_inverse_pair():
    n = 128
    A, Ad = synth.gen_inverse_pair(n, 2)
    hi, lo = O.dd_gemm("N", "N", n, n, n, A, n, Ad, n)
    fp = O.err_stats(O.fp64_gemm("N", "N", n, n, n, A, n, Ad, n), hi, lo)
    errs = {s: O.err_stats(O.dgemm_simple(A, Ad, s), hi, lo) for s in (9, 11, 13)}
    # SPEC S:434 property at s = 11; the paper's claim for INT8xX in general
    assert errs[11]["mean_rel"] < fp["mean_rel"]
    assert errs[13]["mean_rel"] <= errs[11]["mean_rel"] <= errs[9]["mean_rel"]
    assert errs[11]["nw_max"] < fp["nw_max"]
