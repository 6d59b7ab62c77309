"""Pins for the oracle's accuracy-targeted INT8-AUTO (reading A18; Discussion P:713-734: the
loss criterion "does not yield the optimal number of splits ... the accumulation length
should be one of the key factors").

What is pinned, and against what (never against the oracle's own formula):
  * rho_v(t) against the exact relative l1 truncation residual computed with Fractions from
    the definition of a digit (Alg. 4): the oracle's fixed-point value must be an
    upper estimate within the rounding the definition allows;
  * closed forms: vectors exactly representable in t digits have rho(t) = 0; one-element
    vectors; power-of-two scaling, sign and permutation invariance;
  * the inequality the model rests on, |C - C_s|_ij <= sum_t (|R_A(t)| |R_B(s-t)|)_ij, on
    exact rationals (C_s from the oracle's exact integer level sums, C exact);
  * the selection: at the chosen s the SURVEY s8c accuracy gate vs double-double holds, and the
    chosen s equals the survey's FP64-equivalent s within one for the phi sweep;
  * the accumulation length enters: the same data judged with a larger k needs no more slices.
"""
from fractions import Fraction
import math

import numpy as np
import pytest

import oracle as O
import synth


def _E(v):
    mx = max(abs(float(x)) for x in v)
    return math.frexp(mx)[1] if mx else 0


def _trunc(x, E, w, t):
    """First t digits of x (Alg. 4: sgn(x) floor(|x| 2^(wt-E)) 2^(E-wt)) as a Fraction."""
    f = Fraction(abs(x)) * Fraction(2) ** (w * t - E)
    q = f.numerator // f.denominator
    return (1 if x >= 0 else -1) * Fraction(q) * Fraction(2) ** (E - w * t)


def _rho_exact(v, w, t):
    E = _E(v)
    num = sum(abs(Fraction(float(x)) - _trunc(float(x), E, w, t)) for x in v)
    den = sum(abs(Fraction(float(x))) for x in v)
    return num / den


@pytest.mark.parametrize("w", [7, 6, 5])
def test_rho_is_tight_upper_estimate_of_exact_l1_residual(w):
    rng = np.random.default_rng(w)
    V = synth.gen_phi(6, 40, 2.0, 100 + w)
    V[1, :7] = [1.0, -0.5, 2.0 ** -60, 3.0, 5e-324, 1 + 2.0 ** -52, -0.0]
    V[2] *= 2.0 ** -1030            # a row of subnormals and tiny normals
    V[3] = np.ldexp(rng.integers(-1000, 1000, 40).astype(float), 3)  # exact in few digits
    for t in range(0, 12):
        rho = O.trunc_residual(V, 0, 6, 40, 6, w, max(t, 1))
        if t == 0:
            assert rho[0] == 1.0
            continue
        ex = max(_rho_exact(V[r], w, t) for r in range(6))
        got = Fraction(rho[t])
        assert got >= ex * (1 - Fraction(1, 2 ** 52)), (t, float(ex), rho[t])
        # rounding of the fixed-point sums: <= 1 unit of 2^-32 per element on each side, and
        # one rounding of the final division
        slack = []
        for r in range(6):
            v = V[r]
            nrm = sum(abs(Fraction(float(x))) for x in v) * Fraction(2) ** (-_E(v))
            kk = len(v)
            slack.append((_rho_exact(v, w, t) * Fraction(2) ** (w * t) * nrm
                          + Fraction(kk, 2 ** 32)) / (nrm - Fraction(kk, 2 ** 32))
                         * Fraction(2) ** (-w * t))
        assert got <= max(slack) * (1 + Fraction(1, 2 ** 52)), (t, rho[t], float(max(slack)))


def test_rho_closed_forms_and_invariances():
    w = 7
    # exactly representable in 1 digit relative to the row max: rho(t >= 1) = 0
    v = np.array([[0.5, 0.25, -0.375, 2.0 ** -7]])
    rho = O.trunc_residual(v, 0, 1, 4, 1, w, 4)
    assert rho[0] == 1.0 and (rho[1:] == 0).all()
    # 1 + 2^-52 (E = 1): digits hold bits 1..7w below 2^1; the last bit sits at position 53
    x = np.array([[1.0 + 2.0 ** -52]])
    rho = O.trunc_residual(x, 0, 1, 1, 1, w, 9)
    for t in range(1, 10):
        exact = 0.0 if w * t >= 53 else 2.0 ** -52 / (1.0 + 2.0 ** -52)
        assert rho[t] >= exact and (rho[t] == 0) == (exact == 0)
    # power-of-two scaling, sign flips and permutations of a vector do not change rho
    V = synth.gen_phi(3, 50, 1.0, 9)
    base = O.trunc_residual(V, 0, 3, 50, 3, w, 10)
    V2 = np.asfortranarray(-V[:, ::-1] * 2.0 ** 37)
    assert np.array_equal(O.trunc_residual(V2, 0, 3, 50, 3, w, 10), base)
    # both storage orders give the same per-vector statistic
    assert np.array_equal(O.trunc_residual(np.asfortranarray(V.T), 1, 3, 50, 50, w, 10), base)
    # rho is non-increasing in t (more digits never leave more behind)
    assert (np.diff(base) <= 0).all()
    # zero / non-finite vectors are skipped; an all-zero operand has rho = 0 everywhere
    Z = np.zeros((2, 8), order="F")
    assert (O.trunc_residual(Z, 0, 2, 8, 2, w, 5) == 0).all()
    Vn = V.copy(order="F")
    Vn[0, 3] = np.nan
    r_nan = O.trunc_residual(Vn, 0, 3, 50, 3, w, 10)
    r_rest = O.trunc_residual(np.asfortranarray(V[1:]), 0, 2, 50, 2, w, 10)
    assert np.array_equal(r_nan, r_rest)


def test_error_inequality_behind_the_model_exact():
    """|C - C_s|_ij <= sum_{t=0..s} (|R_A(t)| |R_B(s-t)|)_ij on exact rationals (the bound the
    selection's eta estimates); C_s = 2^(E_A+E_B) sum_g L_g 2^-wg from exact level sums."""
    m, n, k = 3, 4, 9
    A = synth.gen_phi(m, k, 2.0, 31)
    B = synth.gen_phi(k, n, 2.0, 32)
    w = O.slice_width(k)
    for s in (1, 2, 3, 5):
        L = O.level_sums("N", "N", m, n, k, A, m, B, k, s)
        for i in range(m):
            EA = _E(A[i])
            RA = [[Fraction(float(A[i, l])) - (_trunc(float(A[i, l]), EA, w, t) if t else 0)
                   for l in range(k)] for t in range(s + 1)]
            for j in range(n):
                EB = _E(B[:, j])
                RB = [[Fraction(float(B[l, j])) - (_trunc(float(B[l, j]), EB, w, t) if t else 0)
                       for l in range(k)] for t in range(s + 1)]
                exact = sum(Fraction(float(A[i, l])) * Fraction(float(B[l, j])) for l in range(k))
                cs = sum(Fraction(int(L[g, i, j])) * Fraction(2) ** (-w * (g + 2))
                         for g in range(s)) * Fraction(2) ** (EA + EB)
                bound = sum(abs(RA[t][l]) * abs(RB[s - t][l]) for t in range(s + 1)
                            for l in range(k))
                assert abs(exact - cs) <= bound, (s, i, j)


@pytest.mark.parametrize("phi_idx,phi,s_eq", [(0, 0.1, 8), (1, 0.5, 9), (2, 1.0, 9),
                                              (3, 2.0, 10)])
def test_selected_s_meets_accuracy_gate(phi_idx, phi, s_eq):
    """At the s the accuracy-targeted AUTO picks (tau = 1) the SURVEY s8c gate vs
    double-double holds (nw_max <= 1e-14, mean_rel <= 1e-14), the pick is the survey's
    FP64-equivalent s within one, and it never exceeds the T = 0 loss pick."""
    m, n, k = 64, 64, 1024
    A = synth.gen_phi(m, k, phi, 201 + phi_idx)
    B = synth.gen_phi(k, n, phi, 211 + phi_idx)
    s, capped = O.auto_splits_acc("N", "N", m, n, k, A, m, B, k, 1.0, 18)
    assert not capped and abs(s - s_eq) <= 1
    assert s <= O.auto_splits("N", "N", m, n, k, A, m, B, k, 0.0, 18)
    C = O.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, np.zeros((m, n), order="F"), m, s)
    hi, lo = O.dd_gemm("N", "N", m, n, k, A, m, B, k)
    st = O.err_stats(C, hi, lo)
    assert st["nw_max"] <= 1e-14 and st["mean_rel"] <= 1e-14, st


def test_accumulation_length_enters_and_tau_orders():
    """A larger k (same element distribution) loosens the FP64 target u sqrt(k) faster than it
    changes the residual statistics; a smaller tau never selects fewer slices; the cap flag."""
    A = synth.gen_phi(32, 256, 1.0, 41)
    B = synth.gen_phi(256, 32, 1.0, 42)
    picks = [O.auto_splits_acc("N", "N", 32, 32, 256, A, 32, B, 256, tau, 18)[0]
             for tau in (1e-4, 1e-2, 1.0, 1e2, 1e4)]
    assert picks == sorted(picks, reverse=True)
    ra = O.trunc_residual(A, 0, 32, 256, 32, O.slice_width(256), 18)
    rb = O.trunc_residual(B, 1, 32, 256, 256, O.slice_width(256), 18)
    eta = [O.acc_eta(ra, rb, s) for s in range(1, 19)]
    assert all(b <= a for a, b in zip(eta, eta[1:]))   # more slices, smaller prediction
    s, capped = O.auto_splits_acc("N", "N", 32, 32, 256, A, 32, B, 256, 1.0, 3)
    assert s == 3 and capped
    # the same rows judged as a longer accumulation (k x 64 by tiling) pick no more slices
    A4 = np.asfortranarray(np.tile(A, (1, 64)))
    B4 = np.asfortranarray(np.tile(B, (64, 1)))
    s1 = O.auto_splits_acc("N", "N", 32, 32, 256, A, 32, B, 256, 1.0, 18)[0]
    s4 = O.auto_splits_acc("N", "N", 32, 32, 256 * 64, A4, 32, B4, 256 * 64, 1.0, 18)[0]
    assert s4 <= s1
