"""Pins for the double-double reference (P:555-560 relative-error metric's C^DD)
against exact rational arithmetic and SPEC worked examples."""
from fractions import Fraction

import numpy as np

import oracle as O
import synth


def test_two_sum_examples():
    assert O.two_sum(1.0, 2.0 ** -53) == (1.0, 2.0 ** -53)
    assert O.two_sum(2.0 ** 52, 1.25) == (2.0 ** 52 + 1, 0.25)
    assert O.two_sum(3.5, 0.0) == (3.5, 0.0)


def test_two_prod_example():
    x = 2.0 ** 27 + 1
    hi, lo = O.two_prod(x, x)
    assert Fraction(hi) + Fraction(lo) == 2 ** 54 + 2 ** 28 + 1
    assert O.two_prod(0.0, 7.0) == (0.0, 0.0)


def test_eft_exactness_random():
    rng = np.random.default_rng(1)
    for _ in range(2000):
        a = float(rng.standard_normal() * 2.0 ** int(rng.integers(-300, 300)))
        b = float(rng.standard_normal() * 2.0 ** int(rng.integers(-300, 300)))
        hi, lo = O.two_sum(a, b)
        assert Fraction(hi) + Fraction(lo) == Fraction(a) + Fraction(b)
        assert hi == a + b
        hi, lo = O.two_prod(a, b)
        assert Fraction(hi) + Fraction(lo) == Fraction(a) * Fraction(b)


def test_dd_gemm_vs_rationals():
    # dd_gemm vs exact rationals < 2^-100 on 8x8 dyadic matrices.
    A = synth.gen_dyadic(8, 8, 40, -30, 30, seed=3)
    B = synth.gen_dyadic(8, 8, 40, -30, 30, seed=4)
    hi, lo = O.dd_gemm("N", "N", 8, 8, 8, A, 8, B, 8)
    for i in range(8):
        for j in range(8):
            ex = sum(Fraction(float(A[i, l])) * Fraction(float(B[l, j])) for l in range(8))
            got = Fraction(hi[i, j]) + Fraction(lo[i, j])
            if ex != 0:
                assert abs(got - ex) / abs(ex) < Fraction(1, 2 ** 100)


def test_dd_gemm_identity_and_transposes():
    B = synth.gen_phi(6, 5, 1.0, seed=7)
    I = np.asfortranarray(np.eye(6))
    hi, lo = O.dd_gemm("N", "N", 6, 5, 6, I, 6, B, 6)
    assert np.array_equal(hi, B) and not lo.any()
    A = synth.gen_phi(4, 9, 1.0, seed=8)
    C = synth.gen_phi(9, 3, 1.0, seed=9)
    h1, l1 = O.dd_gemm("N", "N", 4, 3, 9, A, 4, C, 9)
    h2, l2 = O.dd_gemm("T", "T", 4, 3, 9, np.asfortranarray(A.T), 9, np.asfortranarray(C.T), 3)
    assert np.array_equal(h1, h2) and np.array_equal(l1, l2)


def test_err_stats_zero_for_exact():
    A = synth.gen_int(5, 7, -9, 9, seed=1)
    B = synth.gen_int(7, 4, -9, 9, seed=2)
    hi, lo = O.dd_gemm("N", "N", 5, 4, 7, A, 5, B, 7)
    st = O.err_stats(A @ B, hi, lo)
    assert st["max_rel"] == 0.0 and st["mean_rel"] == 0.0


def _rn(q):
    # round-to-nearest-even of an exact rational: Python's Fraction -> float conversion is
    # correctly rounded (int / int true division), independent of the C code under test
    return float(q)


def test_fp64_gemm_vs_rational_recursive_sum():
    # fp64_gemm_sub (dd_ref.c) is the CPU "DGEMM" of the accuracy-trend pins; its
    # definition: acc_0 = 0, acc_l = RN(acc_{l-1} + RN(x_l * y_l)) in ascending l, no FMA.
    # Checked bit for bit against that recurrence evaluated with exact rationals + one
    # correctly rounded conversion per operation, for all four transpose combinations and a
    # row/column subset.
    m, n, k = 5, 4, 37
    A = synth.gen_phi(m, k, 2.0, seed=21)
    B = synth.gen_phi(k, n, 2.0, seed=22)
    ref = np.zeros((m, n))
    for i in range(m):
        for j in range(n):
            acc = 0.0
            for l in range(k):
                acc = _rn(Fraction(acc) + Fraction(_rn(Fraction(float(A[i, l])) *
                                                        Fraction(float(B[l, j])))))
            ref[i, j] = acc
    got = O.fp64_gemm("N", "N", m, n, k, A, m, B, k)
    assert np.array_equal(got, ref)
    At = np.asfortranarray(A.T)
    Bt = np.asfortranarray(B.T)
    assert np.array_equal(O.fp64_gemm("T", "N", m, n, k, At, k, B, k), ref)
    assert np.array_equal(O.fp64_gemm("N", "T", m, n, k, A, m, Bt, n), ref)
    assert np.array_equal(O.fp64_gemm("T", "T", m, n, k, At, k, Bt, n), ref)
    sub = O.fp64_gemm("N", "N", m, n, k, A, m, B, k, rows=[4, 1], cols=[3, 0, 2])
    assert np.array_equal(sub, ref[np.ix_([4, 1], [3, 0, 2])])
    # the order is recursive (not pairwise): a case where the orders differ
    A1 = np.asfortranarray(np.array([[1.0, 2.0 ** -53, 2.0 ** -53, 2.0 ** -53]]))
    B1 = np.asfortranarray(np.ones((4, 1)))
    assert O.fp64_gemm("N", "N", 1, 1, 4, A1, 1, B1, 4)[0, 0] == 1.0  # each tiny add rounds away
