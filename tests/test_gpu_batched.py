"""GPU parity for the strided-batched entry points (NEXT row f3; quantum-circuit gate
application issues batched cuBLAS GEMMs): every item of the batch is bit-exact
against the oracle on that item, for independent B (strideB > 0), a shared B
(strideB == 0, sliced once), complex operands, and AUTO (num_slices = 0, chosen per item)."""
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


def _stack(mats):
    """Column-major matrices of one shape -> one flat buffer, item b at offset b*stride."""
    return np.concatenate([np.asarray(M).ravel(order="F") for M in mats])


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T")])
@pytest.mark.parametrize("shared_b", [False, True])
def test_dgemm_strided_batched_bitexact(h, ta, tb, shared_b):
    import torch
    m, n, k, s, batch = 48, 37, 150, 9, 5
    As = [synth.gen_phi(*_stored(ta, m, k), 1.0, 10 + b) for b in range(batch)]
    Bs = [synth.gen_phi(*_stored(tb, k, n), 1.0, 20 + (0 if shared_b else b)) for b in range(batch)]
    Cs = [synth.gen_phi(m, n, 1.0, 30 + b) for b in range(batch)]
    sA, sC = As[0].size, m * n
    sB = 0 if shared_b else Bs[0].size
    dA = torch.from_numpy(_stack(As)).cuda()
    dB = torch.from_numpy(_stack(Bs[:1] if shared_b else Bs)).cuda()
    dC = torch.from_numpy(_stack(Cs)).cuda()
    alpha, beta = 1.5, -0.25
    h.dgemm_strided_batched(ta, tb, m, n, k, alpha, dA, As[0].shape[0], sA, dB, Bs[0].shape[0],
                            sB, beta, dC, m, sC, batch, s)
    torch.cuda.synchronize()
    assert h.report()["num_slices"] == s
    got = dC.cpu().numpy()
    for b in range(batch):
        ref = O.dgemm(ta, tb, m, n, k, alpha, As[b], As[b].shape[0], Bs[b], Bs[b].shape[0], beta,
                      Cs[b], m, s)
        gb = np.asfortranarray(got[b * sC:(b + 1) * sC].reshape(n, m).T)
        assert np.array_equal(gb, ref), b


def test_dgemm_strided_batched_auto_per_item(h):
    """num_slices = 0: each item gets the s the oracle's AUTO selects for that item."""
    import torch
    m, n, k, batch = 40, 30, 96, 3
    phis = [0.1, 1.0, 4.0]
    As = [synth.gen_phi(m, k, phis[b], 40 + b) for b in range(batch)]
    Bs = [synth.gen_phi(k, n, phis[b], 50 + b) for b in range(batch)]
    dA, dB = torch.from_numpy(_stack(As)).cuda(), torch.from_numpy(_stack(Bs)).cuda()
    dC = torch.zeros(batch * m * n, dtype=torch.float64, device="cuda")
    h.set_auto(0.0, 20)
    h.dgemm_strided_batched("N", "N", m, n, k, 1.0, dA, m, m * k, dB, k, k * n, 0.0, dC, m,
                            m * n, batch, 0)
    torch.cuda.synchronize()
    got = dC.cpu().numpy()
    for b in range(batch):
        s = O.auto_splits("N", "N", m, n, k, As[b], m, Bs[b], k, 0.0, 20)
        ref = O.dgemm("N", "N", m, n, k, 1.0, As[b], m, Bs[b], k, 0.0,
                      np.zeros((m, n), order="F"), m, s)
        assert np.array_equal(np.asfortranarray(got[b * m * n:(b + 1) * m * n].reshape(n, m).T),
                              ref), b


@pytest.mark.parametrize("shared_b", [False, True])
def test_zgemm_strided_batched_bitexact(h, shared_b):
    """Independent B (op N), or one shared B stored n x k with op(B) = B^H."""
    import torch
    m, n, k, s, batch = 33, 20, 64, 10, 4
    tb = "C" if shared_b else "N"
    As = [synth.gen_phi_complex(m, k, 0.5, 60 + b) for b in range(batch)]
    Bs = [synth.gen_phi_complex(*_stored(tb, k, n), 0.5, 70 + (0 if shared_b else b))
          for b in range(batch)]
    dA = torch.from_numpy(_stack(As)).cuda()
    dB = torch.from_numpy(_stack(Bs[:1] if shared_b else Bs)).cuda()
    dC = torch.zeros(batch * m * n, dtype=torch.complex128, device="cuda")
    ldb = Bs[0].shape[0]
    h.zgemm_strided_batched("N", tb, m, n, k, 1.0 - 0.5j, dA, m, m * k, dB, ldb,
                            0 if shared_b else k * n, 0.0, dC, m, m * n, batch, s)
    torch.cuda.synchronize()
    got = dC.cpu().numpy()
    for b in range(batch):
        ref = O.zgemm("N", tb, m, n, k, 1.0 - 0.5j, As[b], m, Bs[b], ldb, 0.0,
                      np.zeros((m, n), np.complex128, order="F"), m, s)
        gb = np.asfortranarray(got[b * m * n:(b + 1) * m * n].reshape(n, m).T)
        assert np.array_equal(gb, ref), b


def test_batched_edge_cases(h):
    import torch
    import paper_2306_11975_b200 as oz
    d = torch.zeros(16, dtype=torch.float64, device="cuda")
    # batch = 0: no work, success
    h.dgemm_strided_batched("N", "N", 4, 4, 4, 1.0, d, 4, 16, d, 4, 16, 0.0, d, 4, 16, 0, 9)
    # negative stride / batch: invalid value
    with pytest.raises(oz.OzimmuError):
        h.dgemm_strided_batched("N", "N", 4, 4, 4, 1.0, d, 4, -16, d, 4, 16, 0.0, d, 4, 16, 1, 9)
    with pytest.raises(oz.OzimmuError):
        h.dgemm_strided_batched("N", "N", 4, 4, 4, 1.0, d, 4, 16, d, 4, 16, 0.0, d, 4, 16, -1, 9)


def _run_batched_d(h, ta, tb, m, n, k, s, batch, shareA, shareB, alpha, beta, seed):
    import torch
    As = [synth.gen_phi(*_stored(ta, m, k), 1.0, seed + (0 if shareA else b)) for b in range(batch)]
    Bs = [synth.gen_phi(*_stored(tb, k, n), 1.0, seed + 100 + (0 if shareB else b))
          for b in range(batch)]
    Cs = [synth.gen_phi(m, n, 1.0, seed + 200 + b) for b in range(batch)]
    dA = torch.from_numpy(_stack(As[:1] if shareA else As)).cuda()
    dB = torch.from_numpy(_stack(Bs[:1] if shareB else Bs)).cuda()
    dC = torch.from_numpy(_stack(Cs)).cuda()
    h.dgemm_strided_batched(ta, tb, m, n, k, alpha, dA, As[0].shape[0], 0 if shareA else As[0].size,
                            dB, Bs[0].shape[0], 0 if shareB else Bs[0].size, beta, dC, m, m * n,
                            batch, s)
    torch.cuda.synchronize()
    rep = h.report()
    got = dC.cpu().numpy()
    for b in range(batch):
        ref = O.dgemm(ta, tb, m, n, k, alpha, As[b], As[b].shape[0], Bs[b], Bs[b].shape[0], beta,
                      Cs[b], m, s)
        assert np.array_equal(np.asfortranarray(got[b * m * n:(b + 1) * m * n].reshape(n, m).T),
                              ref), b
    return rep


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "T"), ("T", "N"), ("N", "T")])
@pytest.mark.parametrize("share", ["A", "B", "AB"])
def test_fused_batch_bitexact(h, ta, tb, share):
    """Shared-operand batches run as one fused GEMM (<= 5 launches) and stay bit-exact per
    item; m = 16 puts 8 items in one 128-row tile, n = 20 splits items across column tiles."""
    rep = _run_batched_d(h, ta, tb, 16, 20, 96, 8, 37, "A" in share, "B" in share, 1.25, -0.5,
                         300)
    assert rep["launches"] <= 5, rep  # 2 slicing kernels per strided operand + GEMM


def test_fused_batch_large_items(h):
    rep = _run_batched_d(h, "N", "N", 200, 150, 300, 9, 3, False, True, 1.0, 0.0, 400)
    assert rep["launches"] <= 5
    rep = _run_batched_d(h, "N", "N", 150, 200, 300, 9, 3, True, False, 1.0, 0.0, 500)
    assert rep["launches"] <= 5


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("C", "T"), ("T", "C")])
@pytest.mark.parametrize("share", ["A", "B"])
def test_fused_batch_zgemm_bitexact(h, ta, tb, share):
    """Quantum gate application: one 2^d x 2^d gate shared by 2^(N-d-o) state blocks."""
    import torch
    m, n, k, s, batch = 16, 24, 64, 12, 9
    shareA, shareB = share == "A", share == "B"
    As = [synth.gen_phi_complex(*_stored(ta, m, k), 0.5, 600 + (0 if shareA else b))
          for b in range(batch)]
    Bs = [synth.gen_phi_complex(*_stored(tb, k, n), 0.5, 700 + (0 if shareB else b))
          for b in range(batch)]
    Cs = [synth.gen_phi_complex(m, n, 0.5, 800 + b) for b in range(batch)]
    dA = torch.from_numpy(_stack(As[:1] if shareA else As)).cuda()
    dB = torch.from_numpy(_stack(Bs[:1] if shareB else Bs)).cuda()
    dC = torch.from_numpy(_stack(Cs)).cuda()
    alpha, beta = 0.5 + 1.0j, -1.0 + 0.25j
    h.zgemm_strided_batched(ta, tb, m, n, k, alpha, dA, As[0].shape[0], 0 if shareA else As[0].size,
                            dB, Bs[0].shape[0], 0 if shareB else Bs[0].size, beta, dC, m, m * n,
                            batch, s)
    torch.cuda.synchronize()
    assert h.report()["launches"] <= 5
    got = dC.cpu().numpy()
    for b in range(batch):
        ref = O.zgemm(ta, tb, m, n, k, alpha, As[b], As[b].shape[0], Bs[b], Bs[b].shape[0], beta,
                      Cs[b], m, s)
        assert np.array_equal(np.asfortranarray(got[b * m * n:(b + 1) * m * n].reshape(n, m).T),
                              ref), b
