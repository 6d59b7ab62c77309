"""Pins for the oracle's complex GEMM (NEXT row f1; "separating the real and
imaginary parts ... while splitting"; reading A16 in DESIGN.md: real embedding with
interleaved K, one shared exponent per complex row / column)."""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import synth


def test_spec_example_1x1():
    # SPEC oz_zgemm example: (1+2i)(3+4i) = -5+10i exactly with s >= 2.
    C = O.zgemm_simple(np.array([[1 + 2j]]), np.array([[3 + 4j]]), 2)
    assert C[0, 0] == -5 + 10j


def test_small_integer_matrices_exact():
    rng = np.random.default_rng(1)
    A = np.asfortranarray(rng.integers(-50, 51, (7, 11)) + 1j * rng.integers(-50, 51, (7, 11)))
    B = np.asfortranarray(rng.integers(-50, 51, (11, 5)) + 1j * rng.integers(-50, 51, (11, 5)))
    C = O.zgemm_simple(A, B, 4)
    assert np.array_equal(C, A @ B)  # small Gaussian integers: every value exact


def test_real_inputs_reduce_to_dgemm_bitwise():
    """With zero imaginary parts the embedding interleaves zeros: same exponents, same
    digits, same level sums (2k <= 2^17 keeps w) -> Re C equals the real method bitwise."""
    A = synth.gen_phi(9, 40, 1.0, 3)
    B = synth.gen_phi(40, 6, 1.0, 4)
    Cz = O.zgemm_simple(A.astype(np.complex128), B.astype(np.complex128), 9)
    Cd = O.dgemm_simple(A, B, 9)
    assert np.array_equal(Cz.real, Cd) and not Cz.imag.any()


def test_identity_reproduces_A():
    n = 20
    rng = np.random.default_rng(2)
    A = np.asfortranarray((0.5 + 0.5 * rng.random((n, n))) * np.exp(1j * rng.random((n, n))))
    # |Re|,|Im| < 1 with a shared row scale: 9 slices of 7 bits cover the spread
    I = np.asfortranarray(np.eye(n, dtype=np.complex128))
    C = O.zgemm_simple(A, I, 11)
    assert np.max(np.abs(C - A)) <= 2.0 ** -52


@pytest.mark.parametrize("ta,tb", [("T", "N"), ("C", "N"), ("N", "T"), ("N", "C"), ("C", "C")])
def test_transpose_and_conjugate_variants(ta, tb):
    m, n, k = 6, 5, 13
    A = synth.gen_phi_complex(m, k, 0.5, 11)
    B = synth.gen_phi_complex(k, n, 0.5, 12)
    ref = O.zgemm_simple(A, B, 9)
    At = np.asfortranarray(A.T if ta == "T" else A.conj().T)
    Bt = np.asfortranarray(B.T if tb == "T" else B.conj().T)
    a_op = At if ta != "N" else A
    b_op = Bt if tb != "N" else B
    got = O.zgemm_simple(a_op, b_op, 9, transA=ta, transB=tb)
    assert np.array_equal(got, ref)


def test_alpha_beta_formula():
    m, n, k = 5, 4, 9
    A = synth.gen_phi_complex(m, k, 0.5, 21)
    B = synth.gen_phi_complex(k, n, 0.5, 22)
    Cin = synth.gen_phi_complex(m, n, 0.5, 23)
    X = O.zgemm_simple(A, B, 9)
    # alpha = i is exact: i X = -Xim + i Xre; alpha = 2 is exact doubling
    assert np.array_equal(O.zgemm_simple(A, B, 9, alpha_=1j), 1j * X)
    assert np.array_equal(O.zgemm_simple(A, B, 9, alpha_=2.0), 2.0 * X)
    # beta = 0 never reads C (NaN ignored); alpha = 0 never reads A, B
    Cnan = np.full((m, n), np.nan + 1j * np.nan, order="F")
    assert np.array_equal(O.zgemm_simple(A, B, 9, C=Cnan), X)
    assert np.array_equal(O.zgemm_simple(A * np.nan, B, 9, alpha_=0.0, beta=1j, C=Cin), 1j * Cin)
    # general alpha/beta: T = alpha X and U = beta C_in, each part fma(ar, x, -+(ai * y)),
    # then T + U -- re-evaluated with exact rationals and explicit rounding
    al, be = 0.75 - 1.25j, -0.5 + 2.0j
    got = O.zgemm_simple(A, B, 9, alpha_=al, beta=be, C=Cin)

    def cmul(a, x):
        t = float(Fraction(a.imag) * Fraction(x.imag))
        u = float(Fraction(a.imag) * Fraction(x.real))
        re = float(Fraction(a.real) * Fraction(x.real) - Fraction(t))
        im = float(Fraction(a.real) * Fraction(x.imag) + Fraction(u))
        return re, im

    for i in range(m):
        for j in range(n):
            tr, ti = cmul(al, X[i, j])
            ur, ui = cmul(be, Cin[i, j])
            assert got[i, j] == complex(tr + ur, ti + ui)


def test_unitary_product_accuracy():
    # SPEC oz_zgemm example 3: U U^H for a Haar unitary, s = 12 -> off-diagonal < 1e-14.
    U = synth.haar_unitary(16, 5)
    P = O.zgemm_simple(U, U, 12, transB="C")
    off = P - np.diag(np.diag(P))
    assert np.max(np.abs(off)) < 1e-14
    assert np.max(np.abs(np.diag(P) - 1)) < 1e-14


@pytest.mark.parametrize("phi", [0.1, 1.0])
def test_complex_accuracy_vs_dd(phi):
    """Error decays ~2^-7 per slice and saturates below plain FP64 complex GEMM."""
    m = n = 24
    k = 256
    A = synth.gen_phi_complex(m, k, phi, 31)
    B = synth.gen_phi_complex(k, n, phi, 32)
    rh, rl, ih, il = O.dd_zgemm("N", "N", m, n, k, A, m, B, k)
    errs = [O.zerr_stats(O.zgemm_simple(A, B, s), rh, rl, ih, il)["mean_rel"]
            for s in range(3, 12)]
    for a, b in zip(errs[:4], errs[1:5]):
        assert 2 ** 4 < a / b < 2 ** 10
    plain = O.zerr_stats(A @ B, rh, rl, ih, il)["mean_rel"]
    assert errs[-1] <= plain * 1.5 and errs[-1] < 1e-15


def test_dd_zgemm_vs_rationals():
    A = synth.gen_dyadic(4, 6, 30, -20, 20, 1) + 1j * synth.gen_dyadic(4, 6, 30, -20, 20, 2)
    B = synth.gen_dyadic(6, 3, 30, -20, 20, 3) + 1j * synth.gen_dyadic(6, 3, 30, -20, 20, 4)
    A, B = np.asfortranarray(A), np.asfortranarray(B)
    rh, rl, ih, il = O.dd_zgemm("N", "N", 4, 3, 6, A, 4, B, 6)
    for i in range(4):
        for j in range(3):
            er = sum(Fraction(A[i, l].real) * Fraction(B[l, j].real) -
                     Fraction(A[i, l].imag) * Fraction(B[l, j].imag) for l in range(6))
            ei = sum(Fraction(A[i, l].real) * Fraction(B[l, j].imag) +
                     Fraction(A[i, l].imag) * Fraction(B[l, j].real) for l in range(6))
            assert abs(Fraction(rh[i, j]) + Fraction(rl[i, j]) - er) <= abs(er) * Fraction(1, 2 ** 100)
            assert abs(Fraction(ih[i, j]) + Fraction(il[i, j]) - ei) <= abs(ei) * Fraction(1, 2 ** 100)
