"""Pins for the oracle's SplitInt (Alg. 4).

The oracle computes digits with ldexp/floor/fmod; every check below re-derives
the expected value a different way: exact rationals (fractions.Fraction),
integer bit manipulation of the IEEE encoding, or SPEC/paper worked examples."""
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import synth


def _frac_E(row):
    """E with 2^(E-1) <= max|x| < 2^E, by exact rational search (0 for a zero row)."""
    mx = max(abs(Fraction(float(x))) for x in row)
    if mx == 0:
        return 0
    E = 0
    while Fraction(2) ** E <= mx:
        E += 1
    while Fraction(2) ** (E - 1) > mx:
        E -= 1
    return E


def _split_row(row, s, w):
    d, E, bad = O.split(np.asarray(row, dtype=np.float64).reshape(1, -1), 1, 1, len(row),
                        len(row), s, w)
    return d[:, 0, :], int(E[0]), int(bad[0])


def test_spec_examples():
    d, E, _ = _split_row([1.0], 2, 7)
    assert E == 1 and d[:, 0].tolist() == [64, 0]
    d, E, _ = _split_row([3.0, 0.5], 2, 7)
    assert E == 2 and d[0].tolist() == [96, 16] and d[1].tolist() == [0, 0]
    d, E, _ = _split_row([0.0, -0.0, 0.0], 3, 7)
    assert E == 0 and not d.any()


def test_nextafter_one_digits():
    # nextafter(1, 0) = 1 - 2^-53 -> 53 one-bits below 2^0:
    # 7 full digits of 127 then 0b1111000 = 120.
    x = np.nextafter(1.0, 0.0)
    d, E, _ = _split_row([x, -x], 8, 7)
    assert E == 0
    assert d[:, 0].tolist() == [127] * 7 + [120]
    assert d[:, 1].tolist() == [-127] * 7 + [-120]


@pytest.mark.parametrize("phi", [0.1, 1.0, 4.0])
@pytest.mark.parametrize("s,w", [(3, 7), (9, 7), (11, 6), (5, 5)])
def test_reconstruction_is_exact_truncation(phi, s, w):
    """sum_p d_p 2^(E - w p) == sgn(x) * floor(|x| 2^(ws-E)) 2^(E-ws) exactly (Fraction)."""
    M = synth.gen_phi(6, 23, phi, seed=7 + s)
    M[2, 5] = 0.0
    M[3, :] = 0.0
    d, E, _ = O.split(M, 0, 6, 23, 6, s, w)
    for r in range(6):
        assert E[r] == _frac_E(M[r])
        for l in range(23):
            x = Fraction(float(M[r, l]))
            rec = sum(Fraction(int(d[p, r, l])) * Fraction(2) ** (int(E[r]) - w * (p + 1))
                      for p in range(s))
            t = abs(x) * Fraction(2) ** (w * s - int(E[r]))
            expect = (t.numerator // t.denominator) * Fraction(2) ** (int(E[r]) - w * s)
            expect = expect if x >= 0 else -expect
            assert rec == expect, (r, l)
            assert all(abs(int(d[p, r, l])) <= 2 ** w - 1 for p in range(s))
            # sign rule (Alg. 4 line 4): every nonzero digit carries the sign of x
            assert all(int(d[p, r, l]) * (1 if x >= 0 else -1) >= 0 for p in range(s))


def _bits_digits(x, E, s, w):
    """Independent digit extraction from the IEEE-754 bit pattern (integer shifts)."""
    u = struct.unpack("<Q", struct.pack("<d", x))[0]
    neg = u >> 63
    be = (u >> 52) & 0x7FF
    frac = u & ((1 << 52) - 1)
    if be == 0:
        M, e0 = frac, -1074
    else:
        M, e0 = frac | (1 << 52), be - 1075
    out = []
    for p in range(1, s + 1):
        sh = e0 + w * p - E          # |x| 2^(wp - E) = M 2^sh
        v = (M << sh) if sh >= 0 else (M >> (-sh))
        dgt = v & ((1 << w) - 1)
        out.append(-dgt if neg else dgt)
    return out


def test_digits_match_bit_extraction_including_subnormals():
    rng = np.random.default_rng(3)
    rows = []
    rows.append([5e-324, 2.5e-320, -1e-310, 2.2250738585072014e-308, 0.0])       # subnormal maxima
    rows.append([1e300, -3.3e299, 1e-5, 7.0, -1e-300])                          # huge spread
    rows.append(list(rng.standard_normal(5) * 2.0 ** rng.integers(-60, 60, 5)))
    rows.append([1.0, 0.5, 0.25, -2.0 ** -60, 2.0 ** -1073])                    # powers of two
    for s, w in [(8, 7), (16, 7), (20, 5)]:
        for row in rows:
            d, E, _ = _split_row(row, s, w)
            assert E == _frac_E(row)
            for l, x in enumerate(row):
                assert d[:, l].tolist() == _bits_digits(float(x), E, s, w), (row, l)


def test_power_of_two_equivariance():
    M = synth.gen_phi(5, 40, 1.0, seed=11)
    d0, E0, _ = O.split(M, 0, 5, 40, 5, 9, 7)
    for t in (-700, -3, 1, 17, 600):
        d1, E1, _ = O.split(np.ldexp(M, t), 0, 5, 40, 5, 9, 7)
        assert np.array_equal(d0, d1)
        assert np.array_equal(E1, E0 + t)


def test_leading_digit_of_row_max():
    M = synth.gen_phi(32, 64, 2.0, seed=5)
    d, E, _ = O.split(M, 0, 32, 64, 32, 4, 7)
    for r in range(32):
        l = int(np.argmax(np.abs(M[r])))
        assert 64 <= abs(int(d[0, r, l])) <= 127


def test_transposed_access_matches():
    """trans=0 on M equals trans=1 on M^T (same vectors)."""
    M = synth.gen_phi(7, 13, 0.5, seed=2)
    a = O.split(M, 0, 7, 13, 7, 6, 7)
    Mt = np.asfortranarray(M.T)
    b = O.split(Mt, 1, 7, 13, 13, 6, 7)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_nonfinite_rows_flagged():
    M = synth.gen_phi(4, 8, 0.5, seed=9)
    M[1, 3] = np.nan
    M[2, 0] = -np.inf
    d, E, bad = O.split(M, 0, 4, 8, 4, 3, 7)
    assert bad.tolist() == [0, 1, 1, 0]
    assert not d[:, 1, :].any() and not d[:, 2, :].any()
