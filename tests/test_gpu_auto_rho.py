"""GPU parity of the accuracy-targeted INT8-AUTO statistics (reading A18, Discussion
P:713-734): the device rho[t] of one operand (ozimmu_debug_auto_rho: the exact fixed-point
sums N_t, D of every vector, their ratio, the max over the vectors) against the oracle's
oz_ref_trunc_residual, bit for bit, for both vector layouts, the general path (elements more
than 43 bits below their vector's maximum), subnormal-only, zero and NaN/Inf vectors, the three
slice widths and both statistics instances (t <= 12 and t <= 32)."""
import numpy as np
import pytest

import oracle as O
import synth
from gpu_util import dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def h():
    import paper_2306_11975_b200 as oz
    return oz.Handle(0)


def _matrix(shape, seed, special):
    M = synth.gen_phi(*shape, 3.0, seed)
    if special:
        M.flat[::37] *= 2.0 ** -60          # far below the vector maximum: general path
        M.flat[3::101] = 0.0
        M.flat[5::211] = 5e-324
        M.flat[7::89] = -M.flat[7::89]
    return M


def _stored(op, is_rows, rows, kdim):
    if is_rows:
        return (rows, kdim) if op == "N" else (kdim, rows)
    return (kdim, rows) if op == "N" else (rows, kdim)


@pytest.mark.parametrize("op", ["N", "T"])
@pytest.mark.parametrize("is_rows", [1, 0])
@pytest.mark.parametrize("rows,kdim,w,s_max,special", [
    (70, 300, 7, 12, False), (129, 5000, 7, 18, True), (33, 1000, 6, 12, True),
    (8, 20000, 5, 32, True), (300, 64, 7, 32, False)])
def test_rho_bitexact(h, op, is_rows, rows, kdim, w, s_max, special):
    shape = _stored(op, is_rows, rows, kdim)
    M = _matrix(shape, rows * 7 + kdim, special)
    contig = (op != "N") if is_rows else (op == "N")
    ref = O.trunc_residual(M, 1 if contig else 0, rows, kdim, shape[0], w, s_max)
    got = h.debug_auto_rho(op, is_rows, rows, kdim, dev(M), shape[0], w, s_max)
    assert np.array_equal(got, ref), (got, ref)


def test_rho_degenerate_vectors(h):
    rows, kdim = 40, 200
    M = synth.gen_phi(rows, kdim, 1.0, 9)
    M[0, :] = 0.0                                    # all-zero vector: skipped
    M[1, 17] = np.nan                                # NaN vector: skipped
    M[2, :] = np.ldexp(np.abs(M[2, :]), -1060)       # subnormal-only vector
    M[3, 5] = np.inf
    for op in ("N", "T"):
        A = M if op == "N" else np.asfortranarray(M.T)
        ref = O.trunc_residual(A, 0 if op == "N" else 1, rows, kdim, A.shape[0], 7, 16)
        got = h.debug_auto_rho(op, 1, rows, kdim, dev(A), A.shape[0], 7, 16)
        assert np.array_equal(got, ref)
    Z = np.zeros((rows, kdim), order="F")
    assert not h.debug_auto_rho("N", 1, rows, kdim, dev(Z), rows, 7, 12).any()
