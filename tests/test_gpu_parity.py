"""GPU parity: the sm_100a CUDA path (through the C ABI) against the CPU oracle
on identical seeded inputs.  Bar (north_star): exponents, slice planes,
INT32 pair products and level sums bit-exact; C <= 1 ulp (0 ulp expected: both
sides evaluate the same canonical operation sequence)."""
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


def _torch():
    import torch
    return torch


def _stored(trans, rows, cols):
    """Stored shape of an operand whose op() is rows x cols."""
    return (rows, cols) if trans == "N" else (cols, rows)


def run_dgemm(h, ta, tb, m, n, k, alpha, A, B, beta, Cin, s, lda=None, ldb=None, ldc=None):
    lda = lda or A.shape[0]
    ldb = ldb or B.shape[0]
    ldc = ldc or Cin.shape[0]
    dA, dB, dC = dev(A), dev(B), dev(Cin)
    h.dgemm(ta, tb, m, n, k, alpha, dA, lda, dB, ldb, beta, dC, ldc, s)
    _torch().cuda.synchronize()
    return host(dC, Cin.shape[0], Cin.shape[1])


def oracle_dgemm(ta, tb, m, n, k, alpha, A, B, beta, Cin, s, rows=None, cols=None,
                 lda=None, ldb=None, ldc=None):
    return O.dgemm(ta, tb, m, n, k, alpha, A, lda or A.shape[0], B, ldb or B.shape[0], beta,
                   Cin, ldc or Cin.shape[0], s, "L", rows, cols)


# ---------------------------------------------------------------------------------
# A2/A3: exponents and slice planes, bit-exact
# ---------------------------------------------------------------------------------

def _special_matrix(rows, cols, seed):
    M = synth.gen_phi(rows, cols, 2.0, seed)

    def put(i, j, v):
        if isinstance(i, int) and i >= rows:
            return
        if isinstance(j, int) and j >= cols:
            return
        M[i, j] = v

    put(0, slice(None), 0.0)                                 # zero vector (row)
    put(slice(None), 0, 0.0)                                 # zero column
    put(1, slice(1, None, 3), 5e-324)                        # subnormals
    if rows > 2:
        M[2, :] = np.ldexp(np.abs(M[2, :]), -1060)           # row of subnormals only
    put(3, 2, 1e300)                                         # huge spread
    put(4, slice(None), np.nextafter(1.0, 0.0))              # all-127 digits
    put(5, 3, 0.5)                                           # power-of-two maximum
    put(5, slice(0, 3), 0.25)
    put(6, 4, -0.0)
    return M


@pytest.mark.parametrize("op", ["N", "T"])
@pytest.mark.parametrize("is_rows", [1, 0])
@pytest.mark.parametrize("rows,kdim,s", [(77, 333, 9), (130, 64, 13), (9, 1, 3), (256, 2100, 7),
                                         (40, 4097, 17)])
def test_split_bitexact(h, op, is_rows, rows, kdim, s):
    torch = _torch()
    # vector r, element l: A operand: op(M)(r, l); B operand: op(M)(l, r)
    if is_rows:
        shape = (rows, kdim) if op == "N" else (kdim, rows)
    else:
        shape = (kdim, rows) if op == "N" else (rows, kdim)
    M = _special_matrix(*shape, seed=rows + kdim)
    if is_rows:
        d_ref, E_ref, bad = O.split_opA(M, op, rows, kdim, shape[0], s)
    else:
        d_ref, E_ref, bad = O.split_opB(M, op, kdim, rows, shape[0], s)
    planes = empty(s * rows * kdim, torch.int8)
    exps = empty(rows, torch.int32)
    h.debug_split(op, is_rows, rows, kdim, dev(M), shape[0], s, planes, exps)
    torch.cuda.synchronize()
    got = planes.cpu().numpy().reshape(s, rows, kdim)
    E = exps.cpu().numpy()
    assert np.array_equal(E, E_ref)
    assert not bad.any()
    assert np.array_equal(got, d_ref)


def test_split_nonfinite(h):
    torch = _torch()
    M = synth.gen_phi(50, 70, 1.0, 3)
    M[7, 9] = np.nan
    M[20, 0] = np.inf
    M[33, 69] = -np.inf
    d_ref, E_ref, bad = O.split_opA(M, "N", 50, 70, 50, 8)
    planes = empty(8 * 50 * 70, torch.int8)
    exps = empty(50, torch.int32)
    h.debug_split("N", 1, 50, 70, dev(M), 50, 8, planes, exps)
    torch.cuda.synchronize()
    E = exps.cpu().numpy()
    assert np.array_equal(np.where(E == 0x7FFFFFFF, 1, 0), bad.astype(int))
    assert np.array_equal(E[bad == 0], E_ref[bad == 0])
    assert np.array_equal(planes.cpu().numpy().reshape(8, 50, 70), d_ref)


# ---------------------------------------------------------------------------------
# A4: one INT8 x INT8 -> INT32 product on the tcgen05 kernel, bit-exact
# ---------------------------------------------------------------------------------

@pytest.mark.parametrize("m,n,k", [(128, 48, 32), (200, 150, 300), (1, 1, 1), (333, 77, 4100),
                                   (64, 520, 1000)])
def test_pair_product_bitexact(h, m, n, k):
    torch = _torch()
    rng = np.random.default_rng(m * n + k)
    a = rng.integers(-127, 128, (m, k)).astype(np.int8)
    b = rng.integers(-127, 128, (n, k)).astype(np.int8)
    P = empty(m * n, torch.int32)
    h.debug_pair(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), m, n, k, P)
    torch.cuda.synchronize()
    got = P.cpu().numpy().reshape(n, m).T
    ref = O.int_gemm(a, b)
    assert np.array_equal(got, ref)
    # independent library cross-check (cuBLASLt INT8 GEMM) where its shape rules allow
    if m >= 17 and m % 8 == 0 and k % 8 == 0 and n % 8 == 0:
        lib_ref = torch._int_mm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda().t()
                                .contiguous())
        assert np.array_equal(got, lib_ref.cpu().numpy())


def test_pair_product_overflow_edge(h):
    # k = 133144 all-127 digits: 2,147,479,576 <= 2^31 - 1, exact (T5)
    torch = _torch()
    k = 133144
    a = np.full((3, k), 127, np.int8)
    b = np.full((2, k), 127, np.int8)
    b[1] = -127
    P = empty(6, torch.int32)
    h.debug_pair(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), 3, 2, k, P)
    torch.cuda.synchronize()
    got = P.cpu().numpy().reshape(2, 3).T
    assert (got[:, 0] == k * 127 * 127).all() and (got[:, 1] == -k * 127 * 127).all()


# ---------------------------------------------------------------------------------
# A4 + grouping: exact level sums from the fused kernel
# ---------------------------------------------------------------------------------

@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
@pytest.mark.parametrize("m,n,k,s,phi", [(130, 70, 333, 9, 1.0), (64, 64, 64, 7, 0.5),
                                         (257, 97, 1000, 13, 2.0), (1, 1, 1, 3, 0.5)])
def test_level_sums_bitexact(h, ta, tb, m, n, k, s, phi):
    torch = _torch()
    A = synth.gen_phi(*_stored(ta, m, k), phi, 11)
    B = synth.gen_phi(*_stored(tb, k, n), phi, 12)
    out = empty(s * m * n, torch.int64)
    h.debug_level_sums(ta, tb, m, n, k, dev(A), A.shape[0], dev(B), B.shape[0], s, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy().reshape(s, n, m).transpose(0, 2, 1)
    ref = O.level_sums(ta, tb, m, n, k, A, A.shape[0], B, B.shape[0], s)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("k,s", [(16384, 9), (20000, 13), (131072, 9)])
def test_level_sums_multichunk_adversary(h, k, s):
    """K beyond one INT32-safe chunk (s k (2^w-1)^2 > 2^31-1): the kernel's chunked
    drain must stay exact.  Worst case digits (all 127: nextafter(1,0)) plus noise."""
    torch = _torch()
    m, n = 130, 50
    A = np.full((m, k), np.nextafter(1.0, 0.0), order="F")
    A[::3] = synth.gen_phi(len(range(0, m, 3)), k, 0.5, 5)
    B = np.full((k, n), np.nextafter(1.0, 0.0), order="F")
    B[:, 1::4] = -B[:, 1::4]
    out = empty(s * m * n, torch.int64)
    h.debug_level_sums("N", "N", m, n, k, dev(A), m, dev(B), k, s, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy().reshape(s, n, m).transpose(0, 2, 1)
    rows = [0, 1, 2, 64, 127, 128, 129]
    ref = O.level_sums("N", "N", m, n, k, A, m, B, k, s, rows=rows)
    assert np.array_equal(got[:, rows, :], ref)
    rep = h.report()
    # beyond one INT32-safe accumulator: either a second TMEM sub-group region or K chunks
    assert rep["k_chunks"] >= 2 or rep["acc_regions"] == 2, rep
    if k == 16384 and s == 9:
        assert rep["acc_regions"] == 2 and rep["k_chunks"] == 1
    if k == 131072:
        assert rep["k_chunks"] >= 2


# ---------------------------------------------------------------------------------
# Full method: C bit-exact (<= 1 ulp gate) against the oracle
# ---------------------------------------------------------------------------------

@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "C")])
@pytest.mark.parametrize("alpha,beta", [(1.0, 0.0), (-0.5, 2.0), (1.0, 1.0)])
def test_dgemm_c1_config(h, ta, tb, alpha, beta):
    # BASELINE config 1: m = n = k = 64, phi = 0.5, s = 7; seeds 101/102/103
    m = n = k = 64
    s = 7
    A = synth.gen_phi(*_stored(ta, m, k), 0.5, 101)
    B = synth.gen_phi(*_stored(tb, k, n), 0.5, 102)
    Cin = synth.gen_phi(m, n, 0.5, 103)
    got = run_dgemm(h, ta, tb, m, n, k, alpha, A, B, beta, Cin, s)
    ref = oracle_dgemm(ta, tb, m, n, k, alpha, A, B, beta, Cin, s)
    d = ulp_dist(got, ref)
    assert d.max() <= 1
    assert (d == 0).all()


@pytest.mark.parametrize("m,n,k,s", [(1, 1, 1, 1), (1, 300, 17, 9), (300, 1, 17, 9),
                                     (129, 49, 33, 8), (200, 333, 1000, 11), (513, 95, 2049, 16),
                                     (100, 100, 5, 32)])
def test_dgemm_ragged_shapes(h, m, n, k, s):
    A = synth.gen_phi(m, k, 1.0, m + 1)
    B = synth.gen_phi(k, n, 1.0, n + 2)
    Cin = np.zeros((m, n), order="F")
    got = run_dgemm(h, "N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s)
    ref = oracle_dgemm("N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s)
    assert (ulp_dist(got, ref) == 0).all()


def test_dgemm_leading_dimensions(h):
    m, n, k, s = 70, 40, 90, 9
    lda, ldb, ldc = 77, 101, 75
    Abig = synth.gen_phi(lda, k, 0.5, 1)
    Bbig = synth.gen_phi(ldb, n, 0.5, 2)
    Cbig = synth.gen_phi(ldc, n, 0.5, 3)
    got = run_dgemm(h, "N", "N", m, n, k, 1.5, Abig, Bbig, -1.0, Cbig, s, lda, ldb, ldc)
    ref = oracle_dgemm("N", "N", m, n, k, 1.5, Abig, Bbig, -1.0, Cbig, s, lda=lda, ldb=ldb,
                       ldc=ldc)
    assert (ulp_dist(got, ref) == 0).all()
    # rows m..ldc of C untouched
    assert np.array_equal(got[m:], Cbig[m:])


def test_dgemm_edge_values(h):
    m, n, k, s = 40, 30, 50, 9
    A = _special_matrix(m, k, 5)
    B = _special_matrix(k, n, 6).copy(order="F")
    A[10, 10] = 1e-310
    B[3, 7] = 1.7e308
    A[11, :] = 1e200
    B[:, 12] = 1e200                 # overflow to inf in C(11, 12)
    A[12, :] = 1e-200
    B[:, 13] = 1e-200                # underflow into subnormals / zero
    Cin = np.zeros((m, n), order="F")
    got = run_dgemm(h, "N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s)
    ref = oracle_dgemm("N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s)
    assert (ulp_dist(got, ref) == 0).all()
    assert np.isinf(got[11, 12])


def test_dgemm_nonfinite_and_quick_returns(h):
    m, n, k, s = 33, 21, 40, 8
    A = synth.gen_phi(m, k, 0.5, 7)
    B = synth.gen_phi(k, n, 0.5, 8)
    A[4, 5] = np.nan
    B[6, 2] = np.inf
    Cin = np.full((m, n), np.nan, order="F")  # beta = 0: never read
    got = run_dgemm(h, "N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s)
    ref = oracle_dgemm("N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s)
    assert (ulp_dist(got, ref) == 0).all()
    assert np.isnan(got[4]).all() and np.isnan(got[:, 2]).all()
    # alpha = 0: C = beta C, A/B never read (pass NaN matrices)
    C2 = synth.gen_phi(m, n, 0.5, 9)
    got = run_dgemm(h, "N", "N", m, n, k, 0.0, A * np.nan, B, 3.0, C2, s)
    assert np.array_equal(got, 3.0 * C2)
    got = run_dgemm(h, "N", "N", m, n, k, 0.0, A, B, 0.0, Cin, s)
    assert (got == 0).all()
    # k = 0
    got = run_dgemm(h, "N", "N", m, n, 0, 1.0, A, B, 0.5, C2, s)
    assert np.array_equal(got, 0.5 * C2)


@pytest.mark.parametrize("phi_idx,phi", list(enumerate([0.1, 0.5, 1.0, 2.0])))
def test_dgemm_c2_config_sweep(h, phi_idx, phi):
    """BASELINE config 2: 1024^3, phi in {0.1, 0.5, 1, 2}, s = 3..13 (seeds 201+i, 211+i).
    Full GPU result; the oracle on 48 sampled rows x all columns per s."""
    m = n = k = 1024
    A = synth.gen_phi(m, k, phi, 201 + phi_idx)
    B = synth.gen_phi(k, n, phi, 211 + phi_idx)
    Cin = np.zeros((m, n), order="F")
    rows = np.unique(np.concatenate([[0, 1, 127, 128, 1023],
                                     np.random.default_rng(phi_idx).integers(0, m, 43)]))
    for s in range(3, 14):
        got = run_dgemm(h, "N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s)
        ref = oracle_dgemm("N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s, rows=rows)
        assert (ulp_dist(got[rows], ref[rows]) == 0).all(), s


def test_dgemm_determinism_and_row_partition(h):
    """T6 on one GPU: row blocks computed separately (presliced B, as the multi-GPU path
    does) are bitwise identical to the single call; repeated calls are bitwise equal."""
    torch = _torch()
    import paper_2306_11975_b200 as oz
    m, n, k, s = 600, 300, 700, 9
    A = synth.gen_phi(m, k, 1.0, 1)
    B = synth.gen_phi(k, n, 1.0, 2)
    Cin = np.zeros((m, n), order="F")
    full = run_dgemm(h, "N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s)
    again = run_dgemm(h, "N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s)
    assert np.array_equal(full, again)
    bbuf = torch.empty(oz.b_slices_bytes(n, k, s), dtype=torch.uint8, device="cuda")
    h.slice_b("N", k, n, dev(B), k, s, bbuf)
    parts = []
    for r0, r1 in [(0, 150), (150, 400), (400, 600)]:
        Ab = np.asfortranarray(A[r0:r1])
        Cb = torch.zeros((r1 - r0) * n, dtype=torch.float64, device="cuda")
        h.dgemm_presliced_b("N", r1 - r0, n, k, 1.0, dev(Ab), r1 - r0, bbuf, 0.0, Cb, r1 - r0, s)
        torch.cuda.synchronize()
        parts.append(host(Cb, r1 - r0, n))
    assert np.array_equal(np.vstack(parts), full)


def test_row_major_matmul_convenience(h):
    torch = _torch()
    A = synth.gen_phi(90, 70, 0.5, 1)
    B = synth.gen_phi(70, 50, 0.5, 2)
    C = h.matmul(torch.from_numpy(np.ascontiguousarray(A)).cuda(),
                 torch.from_numpy(np.ascontiguousarray(B)).cuda(), 9).cpu().numpy()
    ref = O.dgemm_simple(A, B, 9)
    assert np.array_equal(C, ref)


@pytest.mark.parametrize("size", [8192, 16384])
def test_full_size_sampled(h, size):
    """BASELINE configs 3/4 (8192^3 / 16384^3, phi = 0.5, s = 9) in the launch
    configuration bench.py times; oracle on 24 x 24 sampled output elements."""
    torch = _torch()
    m = n = k = size
    s = 9
    seeds = (301, 302) if size == 8192 else (401, 402)
    A = synth.gen_phi(m, k, 0.5, seeds[0])
    B = synth.gen_phi(k, n, 0.5, seeds[1])
    dA, dB = dev(A), dev(B)
    dC = torch.empty(m * n, dtype=torch.float64, device="cuda")
    h.dgemm("N", "N", m, n, k, 1.0, dA, m, dB, k, 0.0, dC, m, s)
    torch.cuda.synchronize()
    rng = np.random.default_rng(size)
    rows = np.unique(np.concatenate([[0, m - 1, 127, 128], rng.integers(0, m, 20)]))
    cols = np.unique(np.concatenate([[0, n - 1, 47, 48], rng.integers(0, n, 20)]))
    Cs = dC.view(n, m).t()[torch.as_tensor(rows).cuda()][:, torch.as_tensor(cols).cuda()]
    got = Cs.cpu().numpy()
    ref = _oracle_block(A, B, k, s, rows, cols)
    assert (ulp_dist(got, ref) == 0).all()


def _oracle_block(A, B, k, s, rows, cols):
    """Oracle on sampled rows/cols without materialising the full C: the rows of A and
    columns of B are gathered whole (so their exponents are unchanged) and the oracle
    runs on the small problem."""
    As = np.asfortranarray(A[rows, :])
    Bs = np.asfortranarray(B[:, cols])
    C = np.zeros((len(rows), len(cols)), order="F")
    return O.dgemm("N", "N", len(rows), len(cols), k, 1.0, As, len(rows), Bs, k, 0.0, C,
                   len(rows), s)


# ---------------------------------------------------------------------------------
# Accuracy vs double-double and cuBLAS DGEMM (BASELINE metric's max rel err reading)
# ---------------------------------------------------------------------------------

@pytest.mark.parametrize("phi_idx,phi,s_eq", [(0, 0.1, 8), (1, 0.5, 9), (2, 1.0, 9),
                                              (3, 2.0, 10)])
def test_accuracy_gate_vs_dd(h, phi_idx, phi, s_eq):
    """SURVEY s8c gate: nw_max <= 1e-14 and mean_rel <= min(1e-14, cuBLAS DGEMM's), vs DD.
    The smallest passing s (the FP64-equivalent s) must be within one of the survey's."""
    torch = _torch()
    m = n = k = 1024
    A = synth.gen_phi(m, k, phi, 201 + phi_idx)
    B = synth.gen_phi(k, n, phi, 211 + phi_idx)
    rows = np.arange(0, m, 16)
    hi, lo = O.dd_gemm("N", "N", m, n, k, A, m, B, k, rows=rows)
    cub = (torch.from_numpy(A).cuda() @ torch.from_numpy(B).cuda()).cpu().numpy()
    st_cub = O.err_stats(cub[rows], hi, lo)
    Cin = np.zeros((m, n), order="F")
    s_min = None
    for s in range(s_eq - 2, s_eq + 3):
        C = run_dgemm(h, "N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s)
        st = O.err_stats(C[rows], hi, lo)
        if st["nw_max"] <= 1e-14 and st["mean_rel"] <= min(1e-14, st_cub["mean_rel"]):
            s_min = s
            break
    assert s_min is not None and abs(s_min - s_eq) <= 1, (s_min, st_cub)


@pytest.mark.parametrize("cap", [1, 2, 37, 100])
def test_dgemm_capped_grid_bitwise(cap):
    """ozimmu_set_max_sms (persistent grid capped to `cap` SMs, CTA pairs rounded down) gives
    the same bits as the full grid, and 0 restores it."""
    import paper_2306_11975_b200 as oz
    m, n, k, s = 600, 500, 700, 9
    A, B = synth.gen_phi(m, k, 0.5, 71), synth.gen_phi(k, n, 0.5, 72)
    Cin = np.zeros((m, n), order="F")
    h = oz.Handle(0)
    full = run_dgemm(h, "N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s)
    h.set_max_sms(cap)
    capped = run_dgemm(h, "N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s)
    h.set_max_sms(0)
    again = run_dgemm(h, "N", "N", m, n, k, 1.0, A, B, 0.0, Cin, s)
    h.close()
    assert np.array_equal(full, capped) and np.array_equal(full, again)
