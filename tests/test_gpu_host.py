"""GPU parity for ozimmu_dgemm_host (host buffers, copies/slicing/GEMM overlapped in row
blocks of op(A) and column chunks of op(B)): C is bitwise identical to the device-pointer
ozimmu_dgemm and to the oracle (sampled rows/columns straddling every block and chunk
boundary at the pipelined sizes; every element at the small ones), for all transposes,
beta != 0, pinned and pageable memory, INT8-AUTO and the degenerate cases."""
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


def _pinned(M):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(np.asarray(M).ravel(order="F"))).pin_memory()
    return t


def _boundary_idx(total, block):
    idx = {0, total - 1}
    for b in range(block, total, block):
        idx |= {b - 1, b}
    return np.array(sorted(i for i in idx if 0 <= i < total))


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
def test_host_pipelined_bitexact(h, ta, tb):
    import torch
    m, n, k, s = 1300, 1100, 300, 9  # 3 row blocks (512, 512, 276) x 3 column chunks
    A = synth.gen_phi(*_stored(ta, m, k), 1.0, 11)
    B = synth.gen_phi(*_stored(tb, k, n), 1.0, 12)
    Cin = synth.gen_phi(m, n, 1.0, 13)
    alpha, beta = 0.75, -1.5
    hC = _pinned(Cin)
    h.dgemm_host(ta, tb, m, n, k, alpha, _pinned(A), A.shape[0], _pinned(B), B.shape[0], beta,
                 hC, m, s)
    got = np.asfortranarray(hC.numpy().reshape(n, m).T)
    # device-pointer call on the same data
    dC = dev(Cin)
    h.dgemm(ta, tb, m, n, k, alpha, dev(A), A.shape[0], dev(B), B.shape[0], beta, dC, m, s)
    torch.cuda.synchronize()
    assert np.array_equal(got, host(dC, m, n))
    # oracle on rows / columns at every block / chunk boundary
    rows, cols = _boundary_idx(m, 512), _boundary_idx(n, 512)
    ref = O.dgemm(ta, tb, m, n, k, alpha, A, A.shape[0], B, B.shape[0], beta, Cin, m, s,
                  rows=rows, cols=cols)
    assert np.array_equal(got[np.ix_(rows, cols)], ref[np.ix_(rows, cols)])


@pytest.mark.parametrize("m,n", [(2100, 600), (520, 2600)])
def test_host_unequal_block_counts(h, m, n):
    """P row blocks != J column chunks (5 x 2 and 2 x 6): the alternating transfer order
    interleaves them in proportion and every C region is computed exactly once."""
    import torch
    k, s = 200, 9
    A = synth.gen_phi(m, k, 0.5, 31)
    B = synth.gen_phi(k, n, 0.5, 32)
    Cin = synth.gen_phi(m, n, 0.5, 33)
    hC = _pinned(Cin)
    h.dgemm_host("N", "N", m, n, k, 1.25, _pinned(A), m, _pinned(B), k, 0.5, hC, m, s)
    got = np.asfortranarray(hC.numpy().reshape(n, m).T)
    dC = dev(Cin)
    h.dgemm("N", "N", m, n, k, 1.25, dev(A), m, dev(B), k, 0.5, dC, m, s)
    torch.cuda.synchronize()
    assert np.array_equal(got, host(dC, m, n))


@pytest.mark.parametrize("m,n,k,s", [(1, 1, 1, 3), (100, 70, 257, 9), (200, 40, 64, 14)])
def test_host_small_full_oracle(h, m, n, k, s):
    A = synth.gen_phi(m, k, 0.5, m + 1)
    B = synth.gen_phi(k, n, 0.5, n + 2)
    C = np.zeros((m, n), order="F")
    h.dgemm_host("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, s)  # pageable numpy buffers
    ref = O.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, np.zeros((m, n), order="F"), m, s)
    assert np.array_equal(C, ref)


def test_host_ld_padding(h):
    """Leading dimensions larger than the matrices (2-D copies of sub-matrices)."""
    m, n, k, s = 600, 530, 96, 8
    Abig = synth.gen_phi(m + 7, k, 1.0, 21)
    Bbig = synth.gen_phi(k + 5, n, 1.0, 22)
    Cbig = synth.gen_phi(m + 3, n, 1.0, 23)
    C = Cbig.copy(order="F")
    h.dgemm_host("N", "N", m, n, k, 2.0, Abig, m + 7, Bbig, k + 5, 0.5, C, m + 3, s)
    rows, cols = _boundary_idx(m, 512), _boundary_idx(n, 512)
    ref = O.dgemm("N", "N", m, n, k, 2.0, Abig, m + 7, Bbig, k + 5, 0.5, Cbig, m + 3, s,
                  rows=rows, cols=cols)
    assert np.array_equal(C[np.ix_(rows, cols)], ref[np.ix_(rows, cols)])
    # the padding rows of C are untouched
    assert np.array_equal(C[m:], Cbig[m:])


def test_host_auto_and_degenerate(h):
    m, n, k = 90, 60, 128
    A = synth.gen_phi(m, k, 1.0, 31)
    B = synth.gen_phi(k, n, 1.0, 32)
    h.set_auto(0.0, 20)
    C = np.zeros((m, n), order="F")
    h.dgemm_host("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, 0)
    s = O.auto_splits("N", "N", m, n, k, A, m, B, k, 0.0, 20)
    assert h.report()["num_slices"] == s
    ref = O.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, np.zeros((m, n), order="F"), m, s)
    assert np.array_equal(C, ref)
    # alpha = 0: C = beta C (A, B unread)
    Cin = synth.gen_phi(m, n, 1.0, 33)
    C = Cin.copy(order="F")
    h.dgemm_host("N", "N", m, n, k, 0.0, None, m, None, k, -2.0, C, m, 9)
    assert np.array_equal(C, -2.0 * Cin)


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "T"), ("N", "C")])
@pytest.mark.parametrize("T", [0.0, 1.0])
def test_host_auto_pipelined_blocks(h, ta, tb, T):
    """INT8-AUTO through the host pipeline: blocks scanned as they land (8 row blocks x 8
    column chunks), s = the oracle's choice, C bitwise equal to the device-pointer AUTO call."""
    import torch
    m, n, k = 1100, 900, 300
    A = synth.gen_phi(*_stored(ta, m, k), 1.5, 41)
    B = synth.gen_phi(*_stored(tb, k, n), 1.5, 42)
    Cin = synth.gen_phi(m, n, 1.0, 43)
    h.set_auto(T, 20)
    hC = _pinned(Cin)
    h.dgemm_host(ta, tb, m, n, k, 0.5, _pinned(A), A.shape[0], _pinned(B), B.shape[0], 2.0,
                 hC, m, 0)
    s_host = h.report()["num_slices"]
    got = np.asfortranarray(hC.numpy().reshape(n, m).T)
    s_ref = O.auto_splits(ta, tb, m, n, k, A, A.shape[0], B, B.shape[0], T, 20)
    assert s_host == s_ref
    dC = dev(Cin)
    h.dgemm(ta, tb, m, n, k, 0.5, dev(A), A.shape[0], dev(B), B.shape[0], 2.0, dC, m, 0)
    torch.cuda.synchronize()
    assert np.array_equal(got, host(dC, m, n))
    h.set_auto(0.0, 20)
