"""GPU parity over the upper half of the paper's target range, k > 2^17 ("2^11 <=
m, n, k <= 2^20"): the slice width drops to w = 6 (k <= 2^19) and w = 5 (k <= 2^21) by Eq.
alpha with l_acc = 31 (BPS P:457-460; reading A2), so these cases exercise the
W = 6 / 5 slicing instantiations, the w != 7 epilogue scales 2^(-wg) and the K-chunked INT32
budget path (reading A15) that k_oz_gemm takes when one level's s pairs no longer
fit one INT32 accumulator over the whole K.  Small m, n keep the oracle cheap; the shapes still
span two 128-row tiles' worth of ragged edges in n and both storage orders of each operand."""
import numpy as np
import pytest

import oracle as O
import synth
from gpu_util import dev, empty, host, ulp_dist

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def h():
    import paper_2306_11975_b200 as oz
    return oz.Handle(0)


def _stored(trans, rows, cols):
    return (rows, cols) if trans == "N" else (cols, rows)


@pytest.mark.parametrize("k,w", [(2 ** 17 + 1, 6), (2 ** 18, 6), (2 ** 19 + 1, 5), (2 ** 20, 5)])
@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "T")])
def test_dgemm_bigk_bitexact(h, k, w, ta, tb):
    import torch
    m, n, s = 40, 24, 9
    assert O.slice_width(k) == w  # the plan the GPU must follow (A1)
    A = synth.gen_phi(*_stored(ta, m, k), 0.5, 7001 + k % 97)
    B = synth.gen_phi(*_stored(tb, k, n), 0.5, 7002 + k % 89)
    Cin = synth.gen_phi(m, n, 0.5, 7003)
    dA, dB, dC = dev(A), dev(B), dev(Cin)
    h.dgemm(ta, tb, m, n, k, 1.25, dA, A.shape[0], dB, B.shape[0], -0.5, dC, m, s)
    torch.cuda.synchronize()
    rep = h.report()
    assert rep["slice_width"] == w, rep
    # one level's s pairs exceed an INT32 accumulator over the whole K: K chunks or 2 regions
    assert rep["k_chunks"] >= 2 or rep["acc_regions"] == 2, rep
    got = host(dC, m, n)
    ref = O.dgemm(ta, tb, m, n, k, 1.25, A, A.shape[0], B, B.shape[0], -0.5, Cin, m, s)
    assert (ulp_dist(got, ref) == 0).all()


@pytest.mark.parametrize("k,s", [(2 ** 18 + 100, 13), (2 ** 20, 13)])
def test_dgemm_bigk_s13_sampled_rows(h, k, s):
    """s = 13 (91 pair GEMMs) at w = 6 / 5; the oracle on a subset of rows."""
    import torch
    m, n = 40, 24
    A = synth.gen_phi(m, k, 1.0, 7101)
    B = synth.gen_phi(k, n, 1.0, 7102)
    Cin = np.zeros((m, n), order="F")
    dA, dB, dC = dev(A), dev(B), dev(Cin)
    h.dgemm("N", "N", m, n, k, 1.0, dA, m, dB, k, 0.0, dC, m, s)
    torch.cuda.synchronize()
    got = host(dC, m, n)
    rows = [0, 1, 19, 38, 39]
    ref = O.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, Cin, m, s, rows=rows)
    assert (ulp_dist(got[rows], ref[rows]) == 0).all()


@pytest.mark.parametrize("k,w", [(2 ** 18, 6), (2 ** 20, 5)])
def test_split_bigk_bitexact(h, k, w):
    """A2/A3 at w = 6 / 5: exponents and digits of both operand forms, bit-exact."""
    import torch
    rows, s = 5, 11
    M = synth.gen_phi(rows, k, 2.0, 7201)
    M[1, :] = np.nextafter(1.0, 0.0)  # all digits 2^w - 1
    M[2, ::5] = 0.0
    M[3, 7] = 5e-324
    for is_rows, op in ((1, "N"), (1, "T"), (0, "N"), (0, "T")):
        # vector r of the operand = row r of M: A operand rows of op(S), B operand columns
        stored = M if (is_rows == 1) == (op == "N") else M.T
        stored = np.asfortranarray(stored)
        ld = stored.shape[0]
        planes = empty(s * rows * k, torch.int8)
        exps = empty(rows, torch.int32)
        h.debug_split(op, is_rows, rows, k, dev(stored), ld, s, planes, exps)
        torch.cuda.synchronize()
        if is_rows:
            d, E, _ = O.split_opA(stored, op, rows, k, ld, s)
        else:
            d, E, _ = O.split_opB(stored, op, k, rows, ld, s)
        assert np.array_equal(exps.cpu().numpy(), E)
        assert np.array_equal(planes.cpu().numpy().reshape(s, rows, k), d)
    # the all-ones row (53 significant ones) really produces the widest digit of this width
    assert (d[: 53 // w, 1, :] == (1 << w) - 1).all()


def test_level_sums_bigk_adversary(h):
    """Exact int64 level sums at k = 2^19 + 1 (w = 5) with all-maximal digits: every K chunk
    of every pair sits at the INT32 budget the plan computed."""
    import torch
    m, n, k, s = 20, 10, 2 ** 19 + 1, 9
    A = np.full((m, k), np.nextafter(1.0, 0.0), order="F")
    A[::4] = synth.gen_phi(len(range(0, m, 4)), k, 0.5, 7301)
    B = np.full((k, n), np.nextafter(1.0, 0.0), order="F")
    B[:, 1::3] = -B[:, 1::3]
    out = empty(s * m * n, torch.int64)
    h.debug_level_sums("N", "N", m, n, k, dev(A), m, dev(B), k, s, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy().reshape(s, n, m).transpose(0, 2, 1)
    rows = [0, 1, 4, 19]
    ref = O.level_sums("N", "N", m, n, k, A, m, B, k, s, rows=rows)
    assert np.array_equal(got[:, rows, :], ref)
    assert h.report()["k_chunks"] >= 2


def test_dgemm_max_k_supported_and_beyond(h):
    """k = 2^21 (OZIMMU_MAX_K, w = 5) runs and matches the oracle; 2^21 + 1 is UNSUPPORTED."""
    import torch
    import paper_2306_11975_b200 as oz
    m, n, k, s = 3, 5, 2 ** 21, 7
    assert O.slice_width(k) == 5
    A = synth.gen_phi(m, k, 0.5, 7401)
    B = synth.gen_phi(k, n, 0.5, 7402)
    Cin = np.zeros((m, n), order="F")
    dA, dB, dC = dev(A), dev(B), dev(Cin)
    h.dgemm("N", "N", m, n, k, 1.0, dA, m, dB, k, 0.0, dC, m, s)
    torch.cuda.synchronize()
    ref = O.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, Cin, m, s)
    assert (ulp_dist(host(dC, m, n), ref) == 0).all()
    with pytest.raises(oz.OzimmuError) as ei:
        h.dgemm("N", "N", m, n, k + 1, 1.0, dA, m, dB, k + 1, 0.0, dC, m, s)
    assert "UNSUPPORTED" in str(ei.value)


@pytest.mark.parametrize("k,s", [(70000, 9), (140000, 13)])
@pytest.mark.parametrize("ta,tb", [("N", "N"), ("C", "T")])
def test_zgemm_bigk_bitexact(h, k, s, ta, tb):
    """ZGEMM (reading A16: the real embedding has K' = 2k) past 2^17 of K': w = 6 for both
    sizes, the complex slicing forms at W = 6 (both digit windows: s = 9 -> 64 bits, s = 13 ->
    96 bits), and the INT32 budget's K chunks; bitwise vs the oracle."""
    import torch
    m, n = 24, 10
    assert O.slice_width(2 * k) == 6
    A = synth.gen_phi_complex(*_stored(ta, m, k), 0.5, 7101 + k % 31)
    B = synth.gen_phi_complex(*_stored(tb, k, n), 0.5, 7102 + k % 37)
    Cin = synth.gen_phi_complex(m, n, 0.5, 7103)

    def z(a):
        return torch.from_numpy(np.ascontiguousarray(np.asarray(a, np.complex128).ravel(order="F"))).cuda()
    dC = z(Cin)
    h.zgemm(ta, tb, m, n, k, 0.5 - 1.5j, z(A), A.shape[0], z(B), B.shape[0], 0.25j, dC, m, s)
    torch.cuda.synchronize()
    assert h.report()["slice_width"] == 6
    got = dC.cpu().numpy().reshape(n, m).T
    ref = O.zgemm(ta, tb, m, n, k, 0.5 - 1.5j, A, A.shape[0], B, B.shape[0], 0.25j, Cin, m, s)
    assert np.array_equal(got, ref)
