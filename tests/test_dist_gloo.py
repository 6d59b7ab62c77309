"""World-size-2 gloo tests (CPU) of the multi-GPU orchestration in
paper_2306_11975_b200/dist.py: row-block partition, chunked broadcast of the
B-slice buffers from the root, per-chunk GEMM into the local C block.  The math
backend here is a test-only CPU backend over the oracle; the CUDA backend's
per-chunk slicing is covered by tests/test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth
from paper_2306_11975_b200 import dist as D


class OracleBackend:
    """B-slice buffer := the raw float64 columns of op(B)[:, c0:c1] (opaque bytes to the
    orchestration); gemm := the oracle on the local rows and that column block."""

    def b_slices_bytes(self, n, k, s):
        return 8 * n * k

    def alloc(self, nbytes):
        return torch.zeros(nbytes, dtype=torch.uint8)

    def slice_b(self, transB, k, c0, c1, B, ldb, s, buf):
        Bm = np.asarray(B)
        cols = Bm[:k, c0:c1] if transB == "N" else Bm[c0:c1, :k].T
        buf.view(torch.float64).copy_(torch.from_numpy(np.asfortranarray(cols).ravel(order="F")))

    def gemm(self, transA, m_loc, c0, c1, k, alpha, A_loc, lda, buf, beta, C_loc, ldc, s):
        nc = c1 - c0
        Bc = np.asfortranarray(buf.view(torch.float64).numpy().reshape(nc, k).T)
        Cb = np.asfortranarray(C_loc[:m_loc, c0:c1])
        out = O.dgemm(transA, "N", m_loc, nc, k, alpha, A_loc, lda, Bc, k, beta, Cb, m_loc, s)
        C_loc[:m_loc, c0:c1] = out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n, k, s, ta, tb, root, chunk = cfg
        A = synth.gen_phi(*(m, k) if ta == "N" else (k, m), 1.0, 5)
        B = synth.gen_phi(*(k, n) if tb == "N" else (n, k), 1.0, 6)
        Cin = synth.gen_phi(m, n, 0.5, 7)
        r0, r1 = D.row_range(m, world, rank)
        A_loc = np.asfortranarray(A[r0:r1] if ta == "N" else A[:, r0:r1])
        lda = A_loc.shape[0] if A_loc.shape[0] > 0 else 1
        C_loc = np.asfortranarray(Cin[r0:r1]).copy()
        D.dgemm_rowblock(OracleBackend(), ta, tb, r1 - r0, n, k, 1.5, A_loc, lda,
                         B if rank == root else None, B.shape[0], -0.5, C_loc,
                         max(1, r1 - r0), s, root=root, chunk_cols=chunk)
        q.put((rank, r0, r1, C_loc))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [
    (37, 50, 40, 9, "N", "N", 0, 16),
    (64, 33, 100, 7, "T", "N", 1, 8),
    (5, 20, 9, 11, "N", "T", 0, 64),
    (1, 7, 3, 4, "N", "N", 0, 2),   # one rank owns zero rows
])
def test_rowblock_broadcast_matches_single_process(cfg):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    m, n, k, s, ta, tb, root, chunk = cfg
    A = synth.gen_phi(*(m, k) if ta == "N" else (k, m), 1.0, 5)
    B = synth.gen_phi(*(k, n) if tb == "N" else (n, k), 1.0, 6)
    Cin = synth.gen_phi(m, n, 0.5, 7)
    ref = O.dgemm(ta, tb, m, n, k, 1.5, A, A.shape[0], B, B.shape[0], -0.5, Cin, m, s)
    C = np.zeros((m, n))
    for rank, r0, r1, Cl in parts:
        C[r0:r1] = Cl
    assert np.array_equal(C, ref)


def test_row_range_and_chunks():
    for m in (0, 1, 7, 16384):
        for world in (1, 2, 3, 8):
            rr = [D.row_range(m, world, r) for r in range(world)]
            assert rr[0][0] == 0 and rr[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(rr, rr[1:]))
            assert max(r1 - r0 for r0, r1 in rr) - min(r1 - r0 for r0, r1 in rr) <= 1
    assert D.col_chunks(10, 4) == [(0, 4), (4, 8), (8, 10)]
    assert D.col_chunks(0, 4) == []


def _worker2d(rank, world, port, cfg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n, k, s, ta, tb, root, chunk, pr, pc = cfg
        groups = D.make_grid_groups(pr, pc, root)
        A = synth.gen_phi(*(m, k) if ta == "N" else (k, m), 1.0, 15)
        B = synth.gen_phi(*(k, n) if tb == "N" else (n, k), 1.0, 16)
        Cin = synth.gen_phi(m, n, 0.5, 17)
        i, j = D.grid_coords(rank, pr, pc)
        r0, r1 = D.row_range(m, pr, i)
        n0, n1 = D.row_range(n, pc, j)
        A_loc = np.asfortranarray(A[r0:r1] if ta == "N" else A[:, r0:r1])
        lda = A_loc.shape[0] if A_loc.shape[0] > 0 else 1
        C_loc = np.asfortranarray(Cin[r0:r1, n0:n1]).copy()
        D.dgemm_grid2d(OracleBackend(), ta, tb, r1 - r0, n, k, 1.5, A_loc, lda,
                       B if rank == root else None, B.shape[0], -0.5, C_loc, max(1, r1 - r0), s,
                       pr, pc, groups, root=root, chunk_cols=chunk)
        q.put((rank, r0, r1, n0, n1, C_loc))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [
    (37, 50, 40, 9, "N", "N", 0, 16, 2, 2),
    (20, 64, 33, 7, "T", "N", 3, 8, 2, 2),   # root in grid column 1
    (9, 30, 21, 11, "N", "T", 0, 7, 1, 3),   # column blocks only
    (30, 9, 21, 5, "N", "N", 1, 4, 3, 1),    # row blocks only
])
def test_grid2d_broadcast_matches_single_process(cfg):
    m, n, k, s, ta, tb, root, chunk, pr, pc = cfg
    world = pr * pc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker2d, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    A = synth.gen_phi(*(m, k) if ta == "N" else (k, m), 1.0, 15)
    B = synth.gen_phi(*(k, n) if tb == "N" else (n, k), 1.0, 16)
    Cin = synth.gen_phi(m, n, 0.5, 17)
    ref = O.dgemm(ta, tb, m, n, k, 1.5, A, A.shape[0], B, B.shape[0], -0.5, Cin, m, s)
    C = np.full((m, n), np.nan)
    for rank, r0, r1, n0, n1, Cl in parts:
        C[r0:r1, n0:n1] = Cl
    assert np.array_equal(C, ref)
