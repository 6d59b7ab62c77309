"""GPU tests of the library's multi-GPU driver (csrc/dist.cu; C row blocks / 2-D
blocks, op(B) sliced once on the root, its INT8 planes broadcast in column chunks, each chunk's
GEMM waiting only for that chunk, no reduction).

* ozimmu_dgemm_nccl on a real NCCL communicator of one rank (the test boxes have one GPU):
  the whole NCCL code path -- the unique id, ncclCommInitRankConfig with maxCTAs, grouped
  ncclBroadcasts on the collective stream, per-chunk events, the capped GEMM grid -- and the
  result bitwise equal to ozimmu_dgemm, for several chunk widths, both broadcast payloads
  (INT8 planes / FP64 B), all transposes, and the BLAS quick returns.
* ozimmu_dgemm_bcast with 2 and 4 ranks sharing cuda:0 over gloo (NCCL refuses two ranks on
  one device): the same driver with a host-staged broadcast; the assembled C equals the
  single-call result and the CPU oracle bit for bit, row blocks and the 2-D grid."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth

pytestmark = pytest.mark.gpu


def _stored(trans, rows, cols):
    return (rows, cols) if trans == "N" else (cols, rows)


def _flat(X):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(X).ravel(order="F"))).cuda()


def _single(h, ta, tb, m, n, k, alpha, A, B, beta, Cin, s):
    dC = _flat(Cin)
    h.dgemm(ta, tb, m, n, k, alpha, _flat(A), A.shape[0], _flat(B), B.shape[0], beta, dC, m, s)
    torch.cuda.synchronize()
    return dC.cpu().numpy().reshape(n, m).T


@pytest.fixture(scope="module")
def nccl1():
    import paper_2306_11975_b200 as oz
    torch.cuda.set_device(0)
    comm = oz.NcclComm(1, oz.nccl_unique_id(), 0, 0, max_ctas=8)
    h = oz.Handle(0)
    h.set_stream(torch.cuda.current_stream())
    yield h, comm
    torch.cuda.synchronize()
    h.close()
    comm.close()


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "C")])
@pytest.mark.parametrize("chunk,fp64", [(0, False), (96, False), (1000, False), (100, True),
                                        (0, True)])
def test_nccl_one_rank_bitwise(nccl1, ta, tb, chunk, fp64):
    h, comm = nccl1
    m, n, k, s = 300, 1333, 700, 9
    A = synth.gen_phi(*_stored(ta, m, k), 1.0, 1)
    B = synth.gen_phi(*_stored(tb, k, n), 1.0, 2)
    Cin = synth.gen_phi(m, n, 1.0, 3)
    ref = _single(h, ta, tb, m, n, k, 0.75, A, B, 1.25, Cin, s)
    h.set_dist(chunk, 21, fp64)
    dC = _flat(Cin)
    h.dgemm_nccl(comm, 0, ta, tb, m, n, k, 0.75, _flat(A), A.shape[0], _flat(B), B.shape[0],
                 1.25, dC, m, s)
    torch.cuda.synchronize()
    h.set_dist()
    assert np.array_equal(dC.cpu().numpy().reshape(n, m).T, ref)


def test_nccl_one_rank_edges(nccl1):
    import paper_2306_11975_b200 as oz
    h, comm = nccl1
    m, n, k = 130, 250, 200
    A, B = synth.gen_phi(m, k, 0.5, 4), synth.gen_phi(k, n, 0.5, 5)
    Cin = synth.gen_phi(m, n, 0.5, 6)
    # alpha = 0: C = beta C, nothing broadcast, A / B unread
    dC = _flat(Cin)
    h.dgemm_nccl(comm, 0, "N", "N", m, n, k, 0.0, None, m, None, k, -2.0, dC, m, 9)
    torch.cuda.synchronize()
    assert np.array_equal(dC.cpu().numpy().reshape(n, m).T, -2.0 * Cin)
    # a rank without rows only takes part in the broadcasts
    h.dgemm_nccl(comm, 0, "N", "N", 0, n, k, 1.0, None, 1, _flat(B), k, 0.0, None, 1, 9)
    torch.cuda.synchronize()
    # INT8-AUTO cannot be agreed on without A's statistics from every rank
    with pytest.raises(oz.OzimmuError) as ei:
        h.dgemm_nccl(comm, 0, "N", "N", m, n, k, 1.0, _flat(A), m, _flat(B), k, 0.0, dC, m, 0)
    assert "UNSUPPORTED" in str(ei.value)
    with pytest.raises(oz.OzimmuError) as ei:  # root outside the communicator
        h.dgemm_nccl(comm, 1, "N", "N", m, n, k, 1.0, _flat(A), m, _flat(B), k, 0.0, dC, m, 9)
    assert "INVALID" in str(ei.value)
    # large k (w = 6, K chunks in the GEMM) through the driver
    m2, n2, k2 = 40, 200, 2 ** 17 + 3
    A2, B2 = synth.gen_phi(m2, k2, 0.5, 7), synth.gen_phi(k2, n2, 0.5, 8)
    C0 = np.zeros((m2, n2), order="F")
    h.set_dist(96, 8, False)
    dC2 = _flat(C0)
    h.dgemm_nccl(comm, 0, "N", "N", m2, n2, k2, 1.0, _flat(A2), m2, _flat(B2), k2, 0.0, dC2, m2,
                 7)
    torch.cuda.synchronize()
    h.set_dist()
    ref = O.dgemm("N", "N", m2, n2, k2, 1.0, A2, m2, B2, k2, 0.0, C0, m2, 7,
                  rows=[0, 39], cols=list(range(0, n2, 37)))
    got = dC2.cpu().numpy().reshape(n2, m2).T
    cols = list(range(0, n2, 37))
    assert np.array_equal(got[np.ix_([0, 39], cols)], ref[np.ix_([0, 39], cols)])


def test_nccl_graph_and_repeat(nccl1):
    """Back-to-back calls reuse the B-slice buffer: the next call's broadcasts must wait for the
    previous call's GEMMs (ordering through the handle's stream)."""
    h, comm = nccl1
    m, n, k, s = 256, 600, 300, 9
    outs = []
    h.set_dist(128, 8, False)
    for seed in (10, 20, 30):
        A, B = synth.gen_phi(m, k, 1.0, seed), synth.gen_phi(k, n, 1.0, seed + 1)
        dC = torch.empty(m * n, dtype=torch.float64, device="cuda")
        h.dgemm_nccl(comm, 0, "N", "N", m, n, k, 1.0, _flat(A), m, _flat(B), k, 0.0, dC, m, s)
        outs.append((A, B, dC))
    torch.cuda.synchronize()
    h.set_dist()
    for A, B, dC in outs:
        ref = _single(h, "N", "N", m, n, k, 1.0, A, B, 0.0, np.zeros((m, n), order="F"), s)
        assert np.array_equal(dC.cpu().numpy().reshape(n, m).T, ref)


# ---- several ranks on one GPU: the same driver over a gloo broadcast ----------------------

def _free_port():
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    p = sk.getsockname()[1]
    sk.close()
    return p


def _inputs(m, n, k, ta, tb):
    A = synth.gen_phi(*_stored(ta, m, k), 0.5, 11)
    B = synth.gen_phi(*_stored(tb, k, n), 0.5, 12)
    Cin = synth.gen_phi(m, n, 0.5, 13)
    return A, B, Cin


def _worker(rank, world, port, cfg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import paper_2306_11975_b200 as oz
    from paper_2306_11975_b200 import dist as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        m, n, k, s, ta, tb, root, chunk, fp64, pr, pc = cfg
        A, B, Cin = _inputs(m, n, k, ta, tb)
        i, j = D.grid_coords(rank, pr, pc)
        r0, r1 = D.row_range(m, pr, i)
        n0, n1 = D.row_range(n, pc, j)
        ml = r1 - r0
        A_loc = np.asfortranarray(A[r0:r1] if ta == "N" else A[:, r0:r1])
        dA = _flat(A_loc) if ml else None
        dB = _flat(B) if rank == root else None
        dC = _flat(np.asfortranarray(Cin[r0:r1, n0:n1])) if ml else None
        h = oz.Handle(0)
        h.set_stream(torch.cuda.current_stream())
        h.set_dist(chunk, 21, fp64)  # capped GEMM grid (127 SMs) while chunks are in flight
        if pc == 1:
            eng = D.BcastEngine(h)
            D.dgemm_rowblock(eng, ta, tb, ml, n, k, 1.5, dA, max(1, A_loc.shape[0]), dB,
                             B.shape[0], -0.5, dC, max(1, ml), s, root=root)
            calls = eng.calls
        else:
            engines = D.make_grid_engines(lambda g, mem: D.BcastEngine(h, g, mem), pr, pc, root)
            D.dgemm_grid2d(engines, pr, pc, ta, tb, ml, n, k, 1.5, dA, max(1, A_loc.shape[0]),
                           dB, B.shape[0], -0.5, dC, max(1, ml), s, root=root)
            calls = sum(e.calls for e in engines if e is not None)
        torch.cuda.synchronize()
        got = dC.cpu().numpy().reshape(n1 - n0, ml).T.copy() if ml else None
        q.put((rank, r0, r1, n0, n1, got, calls))
        h.close()
    finally:
        dist.destroy_process_group()


def _run(cfg):
    m, n, k, s, ta, tb, root, chunk, fp64, pr, pc = cfg
    world = pr * pc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    A, B, Cin = _inputs(m, n, k, ta, tb)
    C = np.full((m, n), np.nan)
    for rank, r0, r1, n0, n1, Cl, calls in parts:
        if Cl is not None:
            C[r0:r1, n0:n1] = Cl
        assert calls > 0  # every rank took part in the broadcasts
    return A, B, Cin, C


@pytest.mark.parametrize("cfg", [
    (300, 200, 130, 9, "N", "N", 0, 64, False, 2, 1),
    (257, 960, 1000, 7, "T", "N", 1, 96, False, 2, 1),
    (64, 150, 77, 13, "N", "T", 0, 100, False, 2, 1),
    (3, 700, 100, 9, "N", "N", 0, 0, False, 4, 1),      # ranks without rows
    (200, 500, 300, 9, "N", "N", 1, 96, True, 2, 1),    # FP64 broadcast + local slicing
])
def test_rowblock_bcast_driver_bitwise(cfg):
    import paper_2306_11975_b200 as oz
    m, n, k, s, ta, tb = cfg[:6]
    A, B, Cin, C = _run(cfg)
    h = oz.Handle(0)
    one = _single(h, ta, tb, m, n, k, 1.5, A, B, -0.5, Cin, s)
    h.close()
    assert np.array_equal(C, one)
    ref = O.dgemm(ta, tb, m, n, k, 1.5, A, A.shape[0], B, B.shape[0], -0.5, Cin, m, s)
    assert np.array_equal(C, ref)


@pytest.mark.parametrize("cfg", [(300, 260, 130, 9, "N", "N", 0, 64, False, 2, 2),
                                 (200, 150, 500, 13, "T", "T", 3, 48, False, 2, 2)])
def test_grid2d_bcast_driver_bitwise(cfg):
    m, n, k, s, ta, tb = cfg[:6]
    A, B, Cin, C = _run(cfg)
    ref = O.dgemm(ta, tb, m, n, k, 1.5, A, A.shape[0], B, B.shape[0], -0.5, Cin, m, s)
    assert np.array_equal(C, ref)
