"""GPU parity for INT8-AUTO (NEXT row f2, reading A17): the slice count the
device-side mantissa-loss scan selects equals the oracle's, and the AUTO result is
bit-exact against the oracle at that s."""
import numpy as np
import pytest

import oracle as O
import synth
from gpu_util import dev, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def h():
    import paper_2306_11975_b200 as oz
    return oz.Handle(0)


def _stored(trans, rows, cols):
    return (rows, cols) if trans == "N" else (cols, rows)


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
@pytest.mark.parametrize("phi,T", [(0.1, 0.0), (1.0, 0.0), (1.0, 1.0), (2.0, 0.5), (2.0, 4.0)])
def test_auto_dgemm_selects_oracle_s_and_is_bitexact(h, ta, tb, phi, T):
    import torch
    m, n, k = 150, 70, 333
    A = synth.gen_phi(*_stored(ta, m, k), phi, 1)
    B = synth.gen_phi(*_stored(tb, k, n), phi, 2)
    s_ref = O.auto_splits(ta, tb, m, n, k, A, A.shape[0], B, B.shape[0], T, 20)
    h.set_auto(T, 20)
    assert h.auto_splits(ta, tb, m, n, k, dev(A), A.shape[0], dev(B), B.shape[0]) == s_ref
    dC = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    h.dgemm(ta, tb, m, n, k, 1.0, dev(A), A.shape[0], dev(B), B.shape[0], 0.0, dC, m, 0)
    torch.cuda.synchronize()
    assert h.report()["num_slices"] == s_ref
    ref = O.dgemm(ta, tb, m, n, k, 1.0, A, A.shape[0], B, B.shape[0], 0.0,
                  np.zeros((m, n), order="F"), m, s_ref)
    assert np.array_equal(host(dC, m, n), ref)


def test_auto_edge_cases(h):
    m, n, k = 40, 30, 64
    Z = np.zeros((m, k), order="F")
    B = synth.gen_phi(k, n, 1.0, 3)
    h.set_auto(0.0, 16)
    assert h.auto_splits("N", "N", m, n, k, dev(Z), m, dev(np.zeros((k, n), order="F")), k) == 1
    # non-finite rows are excluded from the statistics (their outputs are NaN anyway)
    A = synth.gen_phi(m, k, 1.0, 4)
    A2 = A.copy()
    A2[5, 7] = np.inf
    s_ref = O.auto_splits("N", "N", m, n, k, A2, m, B, k, 0.0, 16)
    assert h.auto_splits("N", "N", m, n, k, dev(A2), m, dev(B), k) == s_ref
    # s_max caps the choice
    h.set_auto(0.0, 3)
    assert h.auto_splits("N", "N", m, n, k, dev(A), m, dev(B), k) == 3
    h.set_auto(0.0, 20)


def _embed(A, B, ta, tb, m, n, k):
    """Reading A16's real operands (plain indexing): A-hat m x 2k, B-hat 2k x 2n."""
    opA = A if ta == "N" else (A.T if ta == "T" else A.conj().T)
    opB = B if tb == "N" else (B.T if tb == "T" else B.conj().T)
    Ah = np.zeros((m, 2 * k))
    Ah[:, 0::2], Ah[:, 1::2] = opA.real, opA.imag
    Bh = np.zeros((2 * k, 2 * n))
    Bh[0::2, 0::2], Bh[1::2, 0::2] = opB.real, -opB.imag
    Bh[0::2, 1::2], Bh[1::2, 1::2] = opB.imag, opB.real
    return np.asfortranarray(Ah), np.asfortranarray(Bh)


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("C", "T")])
def test_auto_zgemm(h, ta, tb):
    import torch
    m, n, k, T = 60, 40, 100, 0.5
    A = synth.gen_phi_complex(*_stored(ta, m, k), 1.0, 5)
    B = synth.gen_phi_complex(*_stored(tb, k, n), 1.0, 6)
    Ah, Bh = _embed(A, B, ta, tb, m, n, k)
    s_ref = O.auto_splits("N", "N", m, 2 * n, 2 * k, Ah, m, Bh, 2 * k, T, 20)
    h.set_auto(T, 20)
    zA = torch.from_numpy(np.ascontiguousarray(A.ravel(order="F"))).cuda()
    zB = torch.from_numpy(np.ascontiguousarray(B.ravel(order="F"))).cuda()
    dC = torch.zeros(m * n, dtype=torch.complex128, device="cuda")
    h.zgemm(ta, tb, m, n, k, 1.0, zA, A.shape[0], zB, B.shape[0], 0.0, dC, m, 0)
    torch.cuda.synchronize()
    assert h.report()["num_slices"] == s_ref
    ref = O.zgemm(ta, tb, m, n, k, 1.0, A, A.shape[0], B, B.shape[0], 0.0,
                  np.zeros((m, n), np.complex128, order="F"), m, s_ref)
    got = dC.cpu().numpy().reshape(n, m).T
    assert np.array_equal(got, ref)
    h.set_auto(0.0, 20)


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "T")])
def test_auto_wide_range_smax32(h, ta, tb):
    """Huge exponent spreads (phi = 8) need many slices; s_max = 32 takes the opt-in
    shared-memory path of the histogram kernels, and T > 0 exercises the F_t - F_l split."""
    m, n, k = 300, 260, 700
    A = synth.gen_phi(*_stored(ta, m, k), 8.0, 81)
    B = synth.gen_phi(*_stored(tb, k, n), 8.0, 82)
    for T in (0.0, 0.5, 3.0, 20.0):
        s_ref = O.auto_splits(ta, tb, m, n, k, A, A.shape[0], B, B.shape[0], T, 32)
        h.set_auto(T, 32)
        assert h.auto_splits(ta, tb, m, n, k, dev(A), A.shape[0], dev(B), B.shape[0]) == s_ref
    h.set_auto(0.0, 20)
