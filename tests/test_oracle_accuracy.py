"""The paper's accuracy trends (s4.2.1, Fig. 6 text) reproduced by the
oracle against the double-double reference.  These pin the whole method's
behaviour, not individual values: a dropped term, a wrong scale or a wrong digit
would break the 2^-7-per-slice decay or the saturation level.

"DGEMM" here is plain binary64 recursive summation on the CPU (oracle/dd_ref.c
fp64_gemm_sub), standing in for cuBLAS; the GPU tests repeat the comparison
against cuBLAS DGEMM."""
import numpy as np
import pytest

import oracle as O
import synth

M = N = 64
K = 1024
S_RANGE = range(3, 14)


@pytest.fixture(scope="module")
def table():
    out = {}
    for idx, phi in enumerate([0.1, 0.5, 1.0, 2.0, 4.0]):
        A = synth.gen_phi(M, K, phi, 201 + idx)
        B = synth.gen_phi(K, N, phi, 211 + idx)
        hi, lo = O.dd_gemm("N", "N", M, N, K, A, M, B, K)
        row = {"dgemm": O.err_stats(O.fp64_gemm("N", "N", M, N, K, A, M, B, K), hi, lo)}
        for s in S_RANGE:
            row[s] = O.err_stats(O.dgemm_simple(A, B, s), hi, lo)
            if s in (9, 11):
                row[("P", s)] = O.err_stats(O.dgemm_simple(A, B, s, mode="P"), hi, lo)
        out[phi] = row
    return out


def test_int8x9_beats_dgemm_at_narrow_range(table):
    # "the error of INT8x9 is smaller than DGEMM when the exponent distribution is narrow (phi = 0.1)"
    r = table[0.1]
    assert r[9]["mean_rel"] < r["dgemm"]["mean_rel"]


def test_int8x9_degrades_with_phi(table):
    # "the error becomes large as the exponent range extends from phi=1 to 4"
    e = [table[phi][9]["mean_rel"] for phi in (0.1, 1.0, 2.0, 4.0)]
    assert e[0] < e[1] < e[2] < e[3]
    assert table[4.0][9]["mean_rel"] > table[4.0]["dgemm"]["mean_rel"]


def test_int8x11_13_match_dgemm_at_wide_range(table):
    # "for INT8x11 and INT8x13, the error is either smaller or almost at the
    # same level as DGEMM, even when ... phi = 4"
    r = table[4.0]
    assert r[13]["mean_rel"] <= r[11]["mean_rel"] <= r[9]["mean_rel"]
    assert r[11]["mean_rel"] <= 2.0 * r["dgemm"]["mean_rel"]
    assert r[13]["mean_rel"] <= r["dgemm"]["mean_rel"]


def test_error_decays_per_slice_then_saturates(table):
    # Each slice adds w = 7 bits of mantissa space: before saturation the
    # mean error drops by roughly 2^-7 per slice.
    for phi, r in table.items():
        e = [r[s]["mean_rel"] for s in S_RANGE]
        for a, b in zip(e, e[1:]):
            assert b <= a * 1.05  # monotone up to rounding noise at saturation
        for s in range(3, 7):
            ratio = r[s]["mean_rel"] / r[s + 1]["mean_rel"]
            assert 2 ** 4 < ratio < 2 ** 10, (phi, s, ratio)
        # saturation: a few ulp of the result
        assert r[13]["mean_rel"] < 1e-15


def test_fp64_equivalent_slice_counts(table):
    # SURVEY s8c gate: nw_max <= 1e-14 and mean_rel <= min(1e-14, DGEMM's).
    def s_eq(phi):
        r = table[phi]
        for s in S_RANGE:
            if r[s]["nw_max"] <= 1e-14 and r[s]["mean_rel"] <= min(1e-14, r["dgemm"]["mean_rel"]):
                return s
        return None
    got = {phi: s_eq(phi) for phi in table}
    # SURVEY s0/A.1 expectations at k = 1024: 8, 9, 9, 10, 11
    assert got[0.1] in (8, 9) and got[0.5] in (8, 9) and got[1.0] == 9
    assert got[2.0] in (9, 10) and got[4.0] in (10, 11)


def test_canonical_order_is_at_least_as_accurate_as_alg3_order(table):
    # Reading A6: mode L (exact level sums, one FP64 add per level) vs mode P
    # (Alg. 3's per-pair FP64 accumulation).
    for phi in table:
        for s in (9, 11):
            assert table[phi][s]["mean_rel"] <= table[phi][("P", s)]["mean_rel"] * 1.05
