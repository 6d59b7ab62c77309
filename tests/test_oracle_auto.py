"""Pins for the oracle's INT8-AUTO split selection (NEXT row f2; "select the
number of splits so that the average mantissa loss in the splitting process is equal to
or smaller than a threshold T"; reading A17).  The loss is re-derived from exact rational
arithmetic (the lowest set bit of |x| and the split's reconstruction), and the selected s
is checked against the split itself."""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import synth


def _frac_loss(x, E, s, w):
    """Loss from first principles: x = odd * 2^e (exact); its significant bits of |x|/2^E
    occupy positions lead .. t_last with t_last = E - e, lead = E - floor(log2|x|)."""
    f = Fraction(abs(x))
    e = 0
    num, den = f.numerator, f.denominator
    # f = num / den with den a power of two: lowest set bit exponent = -log2(den) + v2(num)
    while num % 2 == 0:
        num //= 2
        e += 1
    e -= den.bit_length() - 1
    t_last = E - e
    top = f.numerator.bit_length() - f.denominator.bit_length()  # floor(log2 f) or -1 off
    if Fraction(2) ** top > f:
        top -= 1
    if Fraction(2) ** (top + 1) <= f:
        top += 1
    lead = E - top
    vlen = t_last - lead + 1
    return min(vlen, max(0, t_last - s * w))


def test_loss_definition_vs_rationals():
    rng = np.random.default_rng(0)
    M = synth.gen_phi(4, 30, 2.0, 1)
    M[0, :5] = [1.0, 0.5, 1 + 2.0 ** -52, 3.0, 2.0 ** -40]
    M[1, 2] = 0.0
    w = 7
    for s in (1, 5, 8, 9, 12):
        ls, nnz = O.mantissa_loss(M, 0, 4, 30, 4, w, s)
        total = 0
        cnt = 0
        for r in range(4):
            E = max(np.frexp(np.abs(M[r]))[1])
            for x in M[r]:
                if x != 0:
                    total += _frac_loss(float(x), int(E), s, w)
                    cnt += 1
        assert ls[s - 1] == total and nnz == cnt


def test_zero_loss_iff_split_is_exact():
    """loss_s(x) == 0 exactly when the s digits reconstruct x (no truncation)."""
    M = synth.gen_phi(6, 40, 1.0, 7)
    w = 7
    for s in (6, 8, 10):
        d, E, _ = O.split(M, 0, 6, 40, 6, s, w)
        for r in range(6):
            for l in range(40):
                x = float(M[r, l])
                rec = sum(Fraction(int(d[p, r, l])) * Fraction(2) ** (int(E[r]) - w * (p + 1))
                          for p in range(s))
                exact = rec == Fraction(x)
                assert exact == (_frac_loss(x, int(E[r]), s, w) == 0)


def test_spec_examples():
    # all elements share one exponent (values in [0.5, 1)), w = 7, T = 0 -> s = 8
    A = synth.gen_uniform(10, 50, 0.5, 1.0, 3)
    B = synth.gen_uniform(50, 10, 0.5, 1.0, 4)
    assert O.auto_splits("N", "N", 10, 10, 50, A, 10, B, 50, 0.0) == 8
    # zero matrices -> s = 1
    Z = np.zeros((5, 5), order="F")
    assert O.auto_splits("N", "N", 5, 5, 5, Z, 5, Z, 5, 0.0) == 1


def test_selected_s_is_minimal_and_monotone_in_T():
    A = synth.gen_phi(16, 64, 1.0, 5)
    B = synth.gen_phi(64, 16, 1.0, 6)
    w = O.slice_width(64)
    prev = 99
    for T in (0.0, 0.25, 1.0, 4.0, 16.0):
        s = O.auto_splits("N", "N", 16, 16, 64, A, 16, B, 64, T)
        la, na = O.mantissa_loss(A, 0, 16, 64, 16, w, 32)
        lb, nb = O.mantissa_loss(B, 1, 16, 64, 64, w, 32)
        assert la[s - 1] / na <= T and lb[s - 1] / nb <= T
        if s > 1:
            assert la[s - 2] / na > T or lb[s - 2] / nb > T
        assert s <= prev  # a looser threshold never needs more slices
        prev = s


def test_T0_gives_lossless_splits_and_exact_tiny_products():
    """T = 0: no mantissa loss ("when we set T = 0, no mantissa loss occurs"), so
    every element is reconstructed exactly by its s digits."""
    A = synth.gen_phi(5, 12, 0.5, 9)
    B = synth.gen_phi(12, 4, 0.5, 10)
    s = O.auto_splits("N", "N", 5, 4, 12, A, 5, B, 12, 0.0)
    w = O.slice_width(12)
    for M, trans, rows in ((A, 0, 5), (B, 1, 4)):
        d, E, _ = O.split(M, trans, rows, 12, M.shape[0], s, w)
        for r in range(rows):
            for l in range(12):
                x = float(M[r, l] if trans == 0 else M[l, r])
                rec = sum(Fraction(int(d[p, r, l])) * Fraction(2) ** (int(E[r]) - w * (p + 1))
                          for p in range(s))
                assert rec == Fraction(x)


@pytest.mark.parametrize("phi", [0.1, 1.0, 2.0])
def test_paper_trend_T1_needs_fewer_slices_than_T0(phi):
    # T = 0 picked INT8x12/13, T = 1 picked INT8x8/9 on the circuits
    A = synth.gen_phi(32, 128, phi, 11)
    B = synth.gen_phi(128, 32, phi, 12)
    s0 = O.auto_splits("N", "N", 32, 32, 128, A, 32, B, 128, 0.0)
    s1 = O.auto_splits("N", "N", 32, 32, 128, A, 32, B, 128, 1.0)
    assert s1 < s0
