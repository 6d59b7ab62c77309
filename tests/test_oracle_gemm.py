"""Pins for the oracle's pair products, level sums and FP64 combination
(Alg. 3; readings A6-A9).

Expected values come from: big-integer brute force (Python ints), numpy's
int64 matmul (a library routine the oracle does not use), exact rationals
(fractions.Fraction), the paper's / SPEC's worked examples, and closed-form
error bounds."""
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

U = Fraction(1, 2 ** 53)  # unit roundoff of binary64


def test_int_gemm_spec_example():
    assert O.int_gemm(np.array([[96]], np.int8), np.array([[16]], np.int8)).tolist() == [[1536]]


def test_int_gemm_vs_bigint_and_numpy():
    rng = np.random.default_rng(0)
    a = rng.integers(-127, 128, (5, 37)).astype(np.int8)
    b = rng.integers(-127, 128, (4, 37)).astype(np.int8)
    P = O.int_gemm(a, b)
    for i in range(5):
        for j in range(4):
            assert int(P[i, j]) == sum(int(x) * int(y) for x, y in zip(a[i], b[j]))
    a = rng.integers(-127, 128, (33, 300)).astype(np.int8)
    b = rng.integers(-127, 128, (17, 300)).astype(np.int8)
    assert np.array_equal(O.int_gemm(a, b), a.astype(np.int64) @ b.astype(np.int64).T)


def test_int_gemm_overflow_adversary():
    # 133144 * 127^2 = 2,147,479,576 <= 2^31 - 1: exact; one more term overflows (T5).
    k = 133144
    a = np.full((1, k), 127, np.int8)
    assert int(O.int_gemm(a, a)[0, 0]) == k * 127 * 127
    a = np.full((1, k + 1), 127, np.int8)
    with pytest.raises(OverflowError):
        O.int_gemm(a, a)
    b = np.full((1, k + 1), -127, np.int8)
    with pytest.raises(OverflowError):
        O.int_gemm(a, b)


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
def test_level_sums_vs_numpy(ta, tb):
    m, n, k, s = 9, 7, 50, 5
    A = synth.gen_phi(m if ta == "N" else k, k if ta == "N" else m, 1.0, seed=21)
    B = synth.gen_phi(k if tb == "N" else n, n if tb == "N" else k, 1.0, seed=22)
    w = O.slice_width(k)
    L = O.level_sums(ta, tb, m, n, k, A, A.shape[0], B, B.shape[0], s)
    dA, EA, _ = O.split_opA(A, ta, m, k, A.shape[0], s)
    dB, EB, _ = O.split_opB(B, tb, k, n, B.shape[0], s)
    for g in range(2, s + 2):
        ref = np.zeros((m, n), np.int64)
        for p in range(1, s + 1):
            q = g - p
            if 1 <= q <= s:
                ref += dA[p - 1].astype(np.int64) @ dB[q - 1].astype(np.int64).T
        assert np.array_equal(L[g - 2], ref), g
    # sub-block selection returns the same numbers
    rows, cols = [8, 0, 3], [6, 2]
    Ls = O.level_sums(ta, tb, m, n, k, A, A.shape[0], B, B.shape[0], s, rows, cols)
    assert np.array_equal(Ls, L[:, rows][:, :, cols])
    assert w == 7


def test_one_by_one_spec():
    # 1.5 x 2.5 = 3.75 exactly at s = 2.
    C = O.dgemm_simple(np.array([[1.5]]), np.array([[2.5]]), 2)
    assert C[0, 0] == 3.75


def test_identity_reproduces_B_bitwise():
    # S:390 / SURVEY A.5: A = I, B in [0.5, 1): C == B bitwise once s*w covers
    # offset + 52 bits (s >= 8 at w = 7); s = 7 drops bits.
    n = 24
    B = synth.gen_uniform(n, n, 0.5, 1.0, seed=4)
    I = np.asfortranarray(np.eye(n))
    C8 = O.dgemm_simple(I, B, 8)
    assert np.array_equal(C8, B)
    C7 = O.dgemm_simple(I, B, 7)
    assert not np.array_equal(C7, B)
    assert np.max(np.abs(C7 - B)) <= 2.0 ** -49


def test_integer_matrices_exact():
    A = synth.gen_int(12, 30, -1000, 1000, seed=1)
    B = synth.gen_int(30, 10, -1000, 1000, seed=2)
    exact = A @ B  # small integers: every partial sum exact in binary64
    for s in (3, 5, 9):
        C = O.dgemm_simple(A, B, s)
        if s >= 3:  # 10-bit magnitudes fit in 2 digits of 7 bits -> no dropped pair when s >= 3
            assert np.array_equal(C, exact), s


def _exact_product(A, B, i, j, k):
    return sum(Fraction(float(A[i, l])) * Fraction(float(B[l, j])) for l in range(k))


def _ulp(x):
    x = abs(float(x))
    return np.spacing(x) if x > 0 else 5e-324


@pytest.mark.parametrize("phi", [0.1, 0.5, 1.0, 2.0])
@pytest.mark.parametrize("k", [1, 3, 8, 33])
def test_full_precision_tiny_inputs_vs_rational(phi, k):
    """Tiny inputs with enough slices that no dropped pair is non-zero: the
    triangular sum equals the exact product and mode L is within the recursive-
    summation bound of it; most elements are the correctly rounded value."""
    A = synth.gen_phi(4, k, phi, seed=100 + k)
    B = synth.gen_phi(k, 4, phi, seed=200 + k)
    # s_needed: every element representable in s_needed digits of its row/col scale
    s_need = 1
    for M, rowwise in ((A, True), (B, False)):
        for r in range(4):
            v = M[r] if rowwise else M[:, r]
            E = max(np.frexp(np.abs(v))[1])
            for x in v:
                if x != 0:
                    ex = np.frexp(abs(x))[1] - 1
                    bits = E - ex + 53
                    s_need = max(s_need, -(-bits // 7))
    s = 2 * s_need - 1
    C = O.dgemm_simple(A, B, s)
    L = O.level_sums("N", "N", 4, 4, k, A, 4, B, k, s)
    dA, EA, _ = O.split_opA(A, "N", 4, k, 4, s)
    dB, EB, _ = O.split_opB(B, "N", k, 4, k, s)
    n_exact = 0
    for i in range(4):
        for j in range(4):
            ex = _exact_product(A, B, i, j, k)
            scale = Fraction(2) ** (int(EA[i]) + int(EB[j]))
            tri = sum(Fraction(int(L[g - 2, i, j])) * Fraction(2) ** (-7 * g)
                      for g in range(2, s + 2)) * scale
            assert tri == ex
            bound = (s - 1) * U * sum(abs(Fraction(int(L[g - 2, i, j]))) * Fraction(2) ** (-7 * g)
                                      for g in range(2, s + 2)) * scale
            assert abs(Fraction(float(C[i, j])) - ex) <= bound + Fraction(_ulp(ex)) / 2
            n_exact += float(C[i, j]) == float(ex)
    assert n_exact >= 10  # typically 15-16 of 16 are the correctly rounded product


@pytest.mark.parametrize("mode", ["L", "P"])
def test_truncation_and_rounding_bound_phi(mode):
    """Whole-method bound against the exact rational product (not an oracle value):
    |X - AB| <= 2^(EA+EB) k (s+2) 2^(-ws) + rounding of the combination."""
    m, n, k, s, w = 6, 5, 64, 4, 7
    A = synth.gen_phi(m, k, 1.0, seed=31)
    B = synth.gen_phi(k, n, 1.0, seed=32)
    C = O.dgemm_simple(A, B, s, mode=mode)
    dA, EA, _ = O.split_opA(A, "N", m, k, m, s)
    dB, EB, _ = O.split_opB(B, "N", k, n, k, s)
    for i in range(m):
        for j in range(n):
            ex = _exact_product(A, B, i, j, k)
            sc = Fraction(2) ** (int(EA[i]) + int(EB[j]))
            trunc = sc * k * (s + 2) * Fraction(2) ** (-w * s)
            # sum over kept pairs of |P_pq| 2^(-w(p+q)) (scaled): the magnitude the
            # recursive FP64 summation works on
            absum = sc * sum(Fraction(abs(int((dA[p, i].astype(np.int64) * dB[q, j]).sum())))
                             * Fraction(2) ** (-w * (p + q + 2))
                             for p in range(s) for q in range(s - p))
            rnd = (s * (s + 1) // 2) * U * absum
            assert abs(Fraction(float(C[i, j])) - ex) <= trunc + rnd + Fraction(_ulp(ex)), (i, j)


def test_mode_L_combination_bound_and_order():
    """acc = (((L_{s+1} 2^-w(s+1)) + L_s 2^-ws) + ...) : re-evaluate that exact
    recurrence in rationals with explicit round-to-nearest and compare bitwise."""
    m, n, k, s = 5, 6, 200, 9
    A = synth.gen_phi(m, k, 2.0, seed=41)
    B = synth.gen_phi(k, n, 2.0, seed=42)
    C = O.dgemm_simple(A, B, s)
    L = O.level_sums("N", "N", m, n, k, A, m, B, k, s)
    _, EA, _ = O.split_opA(A, "N", m, k, m, s)
    _, EB, _ = O.split_opB(B, "N", k, n, k, s)
    for i in range(m):
        for j in range(n):
            acc = 0.0
            for g in range(s + 1, 1, -1):
                t = Fraction(int(L[g - 2, i, j])) * Fraction(2) ** (-7 * g)
                acc = float(Fraction(acc) + t)  # float(Fraction) rounds to nearest-even
            X = float(Fraction(acc) * Fraction(2) ** (int(EA[i]) + int(EB[j])))
            assert X == C[i, j]


def test_mode_P_is_alg3_order():
    """Mode P = Alg. 3 lines 4-7 verbatim (i outer, j inner), re-evaluated in rationals."""
    m, n, k, s = 3, 4, 100, 6
    A = synth.gen_phi(m, k, 2.0, seed=51)
    B = synth.gen_phi(k, n, 2.0, seed=52)
    C = O.dgemm_simple(A, B, s, mode="P")
    dA, EA, _ = O.split_opA(A, "N", m, k, m, s)
    dB, EB, _ = O.split_opB(B, "N", k, n, k, s)
    for i in range(m):
        for j in range(n):
            acc = 0.0
            for p in range(1, s + 1):
                for q in range(1, s - p + 2):
                    P = int((dA[p - 1, i].astype(np.int64) * dB[q - 1, j]).sum())
                    acc = float(Fraction(acc) + Fraction(P) * Fraction(2) ** (-7 * (p + q)))
            X = float(Fraction(acc) * Fraction(2) ** (int(EA[i]) + int(EB[j])))
            assert X == C[i, j]


def test_power_of_two_equivariance_of_result():
    A = synth.gen_phi(8, 40, 1.0, seed=61)
    B = synth.gen_phi(40, 6, 1.0, seed=62)
    C = O.dgemm_simple(A, B, 7)
    C2 = O.dgemm_simple(np.ldexp(A, 13), np.ldexp(B, -40), 7)
    assert np.array_equal(np.ldexp(C, -27), C2)


def test_transpose_variants_agree():
    m, n, k = 7, 5, 33
    A = synth.gen_phi(m, k, 0.5, seed=71)
    B = synth.gen_phi(k, n, 0.5, seed=72)
    ref = O.dgemm_simple(A, B, 8)
    At, Bt = np.asfortranarray(A.T), np.asfortranarray(B.T)
    assert np.array_equal(O.dgemm_simple(At, B, 8, transA="T"), ref)
    assert np.array_equal(O.dgemm_simple(A, Bt, 8, transB="T"), ref)
    assert np.array_equal(O.dgemm_simple(At, Bt, 8, transA="T", transB="C"), ref)
    # row-major trick: C^T = B^T A^T gives the transposed result bitwise (exponents symmetric)
    CT = O.dgemm_simple(Bt, At, 8)
    assert np.array_equal(CT.T, ref)


def test_alpha_beta_semantics():
    m, n, k = 4, 3, 10
    A = synth.gen_phi(m, k, 0.5, seed=81)
    B = synth.gen_phi(k, n, 0.5, seed=82)
    Cin = synth.gen_phi(m, n, 0.5, seed=83)
    X = O.dgemm_simple(A, B, 9)
    C = O.dgemm_simple(A, B, 9, alpha_=-0.5, beta=2.0, C=Cin)
    # fma(alpha, X, beta*C_in): beta*C_in rounded first, then one rounding of the fma
    expect = [[float(Fraction(-0.5) * Fraction(float(X[i, j])) + Fraction(float(2.0 * Cin[i, j])))
               for j in range(n)] for i in range(m)]
    assert np.array_equal(C, np.array(expect))
    # beta = 0: C_in not read (NaN ignored)
    Cnan = np.full((m, n), np.nan, order="F")
    C = O.dgemm_simple(A, B, 9, alpha_=3.0, beta=0.0, C=Cnan)
    assert np.array_equal(C, 3.0 * X)
    # alpha = 0: A, B not read
    Anan = np.full_like(A, np.nan)
    C = O.dgemm_simple(Anan, B, 9, alpha_=0.0, beta=2.0, C=Cin)
    assert np.array_equal(C, 2.0 * Cin)
    C = O.dgemm_simple(Anan, B, 9, alpha_=0.0, beta=0.0, C=Cnan)
    assert np.array_equal(C, np.zeros((m, n)))


def test_nonfinite_propagation():
    m, n, k = 5, 4, 12
    A = synth.gen_phi(m, k, 0.5, seed=91)
    B = synth.gen_phi(k, n, 0.5, seed=92)
    A[2, 7] = np.inf
    B[3, 1] = np.nan
    C = O.dgemm_simple(A, B, 8)
    bad = np.isnan(C)
    assert bad[2, :].all() and bad[:, 1].all()
    assert bad.sum() == n + m - 1
    A2, B2 = A.copy(), B.copy()
    A2[2, 7] = 0.0
    B2[3, 1] = 0.0
    ok = O.dgemm_simple(A2, B2, 8)
    # every other element only depends on finite rows / columns: unchanged
    rows = [0, 1, 3, 4]
    cols = [0, 2, 3]
    assert np.array_equal(C[np.ix_(rows, cols)], ok[np.ix_(rows, cols)])


def test_zero_and_signed_zero():
    A = np.zeros((3, 4), order="F")
    B = synth.gen_phi(4, 2, 0.5, seed=1)
    C = O.dgemm_simple(A, B, 5)
    assert np.array_equal(C, np.zeros((3, 2))) and not np.signbit(C).any()
    C = O.dgemm_simple(A, B, 5, alpha_=-1.0)
    assert (C == 0).all()  # -0.0 by IEEE; compared as equal


def test_subblock_equals_full():
    m, n, k = 20, 11, 70
    A = synth.gen_phi(m, k, 1.0, seed=5)
    B = synth.gen_phi(k, n, 1.0, seed=6)
    full = O.dgemm_simple(A, B, 9)
    rows, cols = [19, 0, 7], [10, 3]
    sub = O.dgemm_simple(A, B, 9, rows=rows, cols=cols)
    assert np.array_equal(sub[np.ix_(rows, cols)], full[np.ix_(rows, cols)])


def test_oracle_deterministic_across_thread_counts():
    """the oracle parallelises over (i, j) only, so every element's operation
    sequence -- and the bits of C -- must not depend on OMP_NUM_THREADS."""
    import hashlib
    import subprocess
    import sys
    code = ("import sys, hashlib, numpy as np; sys.path.insert(0, %r); import oracle as O, synth;"
            "A = synth.gen_phi(70, 300, 1.0, 81); B = synth.gen_phi(300, 50, 1.0, 82);"
            "C = synth.gen_phi(70, 50, 1.0, 83);"
            "R = O.dgemm('N', 'N', 70, 50, 300, 0.5, A, 70, B, 300, -1.5, C, 70, 9);"
            "print(hashlib.sha1(np.ascontiguousarray(R).tobytes()).hexdigest())") % ROOT
    out = []
    for th in ("1", "3", "8"):
        env = dict(os.environ, OMP_NUM_THREADS=th)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           timeout=120)
        assert r.returncode == 0, r.stderr[-2000:]
        out.append(r.stdout.strip())
    assert len(set(out)) == 1, out
