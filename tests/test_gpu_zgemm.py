"""GPU parity for ozimmu_zgemm (NEXT row f1) against the complex oracle (reading A16):
bit-exact C on identical seeded inputs, all op combinations, ragged shapes, complex
alpha/beta, the INT32-budget edge (k = 2^16 -> K' = 2^17), the quantum-circuit shapes of
BASELINE config 5 (sampled), and accuracy vs the double-double complex reference."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def h():
    import paper_2306_11975_b200 as oz
    return oz.Handle(0)


def zdev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.complex128).ravel(order="F"))).cuda()


def zhost(t, rows, cols):
    x = t.cpu().numpy()
    return np.asfortranarray(x[: rows * cols].reshape((cols, rows)).T)


def _stored(trans, rows, cols):
    return (rows, cols) if trans == "N" else (cols, rows)


def run_z(h, ta, tb, m, n, k, alpha, A, B, beta, Cin, s):
    import torch
    dC = zdev(Cin)
    h.zgemm(ta, tb, m, n, k, alpha, zdev(A), A.shape[0], zdev(B), B.shape[0], beta, dC,
            Cin.shape[0], s)
    torch.cuda.synchronize()
    return zhost(dC, Cin.shape[0], Cin.shape[1])


@pytest.mark.parametrize("ta", ["N", "T", "C"])
@pytest.mark.parametrize("tb", ["N", "T", "C"])
def test_zgemm_ops_bitexact(h, ta, tb):
    m, n, k, s = 70, 45, 131, 9
    A = synth.gen_phi_complex(*_stored(ta, m, k), 0.5, 1)
    B = synth.gen_phi_complex(*_stored(tb, k, n), 0.5, 2)
    Cin = synth.gen_phi_complex(m, n, 0.5, 3)
    for alpha, beta in [(1.0, 0.0), (0.75 - 1.25j, -0.5 + 2.0j)]:
        got = run_z(h, ta, tb, m, n, k, alpha, A, B, beta, Cin, s)
        ref = O.zgemm(ta, tb, m, n, k, alpha, A, A.shape[0], B, B.shape[0], beta, Cin, m, s)
        assert np.array_equal(got, ref), (alpha, beta)


@pytest.mark.parametrize("m,n,k,s", [(1, 1, 1, 2), (129, 33, 7, 12), (200, 97, 1000, 8),
                                     (64, 130, 300, 13), (17, 5, 64, 20)])
def test_zgemm_ragged_bitexact(h, m, n, k, s):
    A = synth.gen_phi_complex(m, k, 1.0, m + 7)
    B = synth.gen_phi_complex(k, n, 1.0, n + 8)
    Cin = np.zeros((m, n), dtype=np.complex128, order="F")
    got = run_z(h, "N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s)
    ref = O.zgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, Cin, m, s)
    assert np.array_equal(got, ref)


def test_zgemm_real_inputs_equal_dgemm(h):
    import torch
    m, n, k, s = 90, 60, 200, 9
    A = synth.gen_phi(m, k, 1.0, 1)
    B = synth.gen_phi(k, n, 1.0, 2)
    got = run_z(h, "N", "N", m, n, k, 1.0, A.astype(np.complex128), B.astype(np.complex128),
                0.0, np.zeros((m, n), np.complex128, order="F"), s)
    dA = torch.from_numpy(A.ravel(order="F").copy()).cuda()
    dB = torch.from_numpy(B.ravel(order="F").copy()).cuda()
    dC = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    h.dgemm("N", "N", m, n, k, 1.0, dA, m, dB, k, 0.0, dC, m, s)
    torch.cuda.synchronize()
    real = dC.cpu().numpy().reshape(n, m).T
    assert np.array_equal(got.real, real) and not got.imag.any()


def test_zgemm_budget_edge_k65536(h):
    """k = 2^16 -> K' = 2^17: w = 7 at the INT32 limit; the top levels need a second TMEM
    region or K chunks (k up to 2^16 is BASELINE config 5's range)."""
    m, n, k, s = 40, 24, 65536, 9
    A = synth.gen_phi_complex(m, k, 0.5, 11)
    B = synth.gen_phi_complex(k, n, 0.5, 12)
    got = run_z(h, "N", "N", m, n, k, 1.0, A, B, 0.0, np.zeros((m, n), np.complex128, order="F"), s)
    rows = [0, 17, 39]
    ref = O.zgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0,
                  np.zeros((m, n), np.complex128, order="F"), m, s, rows=rows)
    assert np.array_equal(got[rows], ref[rows])
    assert h.report()["k_chunks"] >= 2 or h.report()["acc_regions"] == 2


def test_zgemm_nonfinite_and_quick_returns(h):
    m, n, k, s = 20, 15, 30, 9
    A = synth.gen_phi_complex(m, k, 0.5, 21)
    B = synth.gen_phi_complex(k, n, 0.5, 22)
    A[3, 4] = complex(np.nan, 0.0)
    B[5, 6] = complex(0.0, np.inf)
    Cin = np.full((m, n), np.nan, dtype=np.complex128, order="F")
    got = run_z(h, "N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s)
    ref = O.zgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, Cin, m, s)
    same = (got == ref) | (np.isnan(got.real) & np.isnan(ref.real))
    assert same.all()
    assert np.isnan(got[3]).all() and np.isnan(got[:, 6]).all()
    C2 = synth.gen_phi_complex(m, n, 0.5, 23)
    got = run_z(h, "N", "N", m, n, k, 0.0, A, B, 1j, C2, s)
    assert np.array_equal(got, O.zgemm("N", "N", m, n, k, 0.0, A, m, B, k, 1j, C2, m, s))


@pytest.mark.parametrize("d", [8, 10])
def test_quantum_circuit_shapes_sampled(h, d):
    """BASELINE config 5 shape family: matmul-(2^(N-d), 2^d, 2^d) with a Haar gate
    U applied to a normalised random state; N = 20 here (the full N = 28 state,
    4 GiB, is a benchmark size)."""
    N = 20
    m, n = 2 ** (N - d), 2 ** d
    psi = synth.gen_phi_complex(m, n, 0.1, 31)
    psi /= np.linalg.norm(psi)
    U = synth.haar_unitary(n, 32)
    got = run_z(h, "N", "T", m, n, n, 1.0, psi, U, 0.0, np.zeros((m, n), np.complex128, order="F"), 12)
    rows = np.random.default_rng(d).integers(0, m, 12)
    ref = O.zgemm("N", "T", m, n, n, 1.0, psi, m, U, n, 0.0,
                  np.zeros((m, n), np.complex128, order="F"), m, 12, rows=rows)
    assert np.array_equal(got[rows], ref[rows])
    # norm preserved to FP64 accuracy (U unitary)
    assert abs(np.linalg.norm(got) - 1.0) < 1e-13


def test_zgemm_accuracy_vs_dd(h):
    import torch
    m = n = k = 512
    A = synth.gen_phi_complex(m, k, 0.5, 41)
    B = synth.gen_phi_complex(k, n, 0.5, 42)
    rows = np.arange(0, m, 16)
    rh, rl, ih, il = O.dd_zgemm("N", "N", m, n, k, A, m, B, k, rows=rows)
    cub = (torch.from_numpy(A).cuda() @ torch.from_numpy(B).cuda()).cpu().numpy()
    st_cub = O.zerr_stats(cub[rows], rh, rl, ih, il)
    got = run_z(h, "N", "N", m, n, k, 1.0, A, B, 0.0, np.zeros((m, n), np.complex128, order="F"), 10)
    st = O.zerr_stats(got[rows], rh, rl, ih, il)
    assert st["nw_max"] <= 1e-14 and st["mean_rel"] <= min(1e-14, st_cub["mean_rel"]), (st, st_cub)
