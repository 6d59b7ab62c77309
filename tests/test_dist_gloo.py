"""World-size 2-4 gloo tests (CPU) of the multi-GPU orchestration in
paper_2306_11975_b200/dist.py: row-block partition, the 2-D grid with its
per-column broadcast groups, the order in which ranks enter the groups (the root takes part in
every group), and that the assembled C equals the single-process oracle result bit for bit.
The library's own chunked broadcast / per-chunk GEMM driver (csrc/dist.cu) runs on the GPU in
tests/test_gpu_dist.py; here an oracle-backed engine stands in for it with the same protocol:
op(B) (this engine sends its FP64 columns) goes from the group's root to every member, each
member computes its own rows."""
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


class OracleEngine:
    """Test engine with the library driver's interface: the root broadcasts op(B) (k x n,
    FP64) inside the group, every member runs the oracle on its rows."""

    def __init__(self, group=None, members=None):
        self.group = group
        self.members = members if members is not None else list(range(dist.get_world_size()))
        self.me = self.members.index(dist.get_rank())

    def dgemm(self, root, transA, transB, m_loc, n, k, alpha, A_loc, lda, B, ldb, beta, C_loc,
              ldc, s):
        buf = torch.zeros(k * n, dtype=torch.float64)
        if self.me == root:
            opB = np.asarray(B)[:k, :n] if transB == "N" else np.asarray(B)[:n, :k].T
            buf.copy_(torch.from_numpy(np.asfortranarray(opB).ravel(order="F")))
        if len(self.members) > 1:
            dist.broadcast(buf, src=self.members[root], group=self.group)
        if m_loc == 0:
            return
        Bc = np.asfortranarray(buf.numpy().reshape(n, k).T)
        C_loc[:m_loc, :n] = O.dgemm(transA, "N", m_loc, n, k, alpha, A_loc, lda, Bc, k, beta,
                                    np.asfortranarray(C_loc[:m_loc, :n]), m_loc, s)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(m, n, k, ta, tb, seed):
    A = synth.gen_phi(*(m, k) if ta == "N" else (k, m), 1.0, seed)
    B = synth.gen_phi(*(k, n) if tb == "N" else (n, k), 1.0, seed + 1)
    Cin = synth.gen_phi(m, n, 0.5, seed + 2)
    return A, B, Cin


def _worker(rank, world, port, cfg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n, k, s, ta, tb, root = cfg
        A, B, Cin = _inputs(m, n, k, ta, tb, 5)
        r0, r1 = D.row_range(m, world, rank)
        A_loc = np.asfortranarray(A[r0:r1] if ta == "N" else A[:, r0:r1])
        lda = A_loc.shape[0] if A_loc.shape[0] > 0 else 1
        C_loc = np.asfortranarray(Cin[r0:r1]).copy()
        D.dgemm_rowblock(OracleEngine(), ta, tb, r1 - r0, n, k, 1.5, A_loc, lda,
                         B if rank == root else None, B.shape[0], -0.5, C_loc,
                         max(1, r1 - r0), s, root=root)
        q.put((rank, r0, r1, C_loc))
    finally:
        dist.destroy_process_group()


def _spawn(target, world, cfg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return parts


@pytest.mark.parametrize("cfg", [
    (37, 50, 40, 9, "N", "N", 0),
    (64, 33, 100, 7, "T", "N", 1),
    (5, 20, 9, 11, "N", "T", 0),
    (1, 7, 3, 4, "N", "N", 0),   # one rank owns zero rows
])
def test_rowblock_broadcast_matches_single_process(cfg):
    world = 2
    parts = _spawn(_worker, world, cfg)
    m, n, k, s, ta, tb, root = cfg
    A, B, Cin = _inputs(m, n, k, ta, tb, 5)
    ref = O.dgemm(ta, tb, m, n, k, 1.5, A, A.shape[0], B, B.shape[0], -0.5, Cin, m, s)
    C = np.zeros((m, n))
    for rank, r0, r1, Cl in parts:
        C[r0:r1] = Cl
    assert np.array_equal(C, ref)


def test_row_range_and_grid_members():
    for m in (0, 1, 7, 16384):
        for world in (1, 2, 3, 8):
            rr = [D.row_range(m, world, r) for r in range(world)]
            assert rr[0][0] == 0 and rr[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(rr, rr[1:]))
            assert max(r1 - r0 for r0, r1 in rr) - min(r1 - r0 for r0, r1 in rr) <= 1
    # 2 x 4 grid, root 0: column j's group = root + column j
    assert D.grid_members(2, 4, 0, 0) == [0, 4]
    assert D.grid_members(2, 4, 0, 3) == [0, 3, 7]
    assert D.grid_members(2, 2, 3, 0) == [0, 2, 3]
    assert [D.grid_coords(r, 2, 4) for r in (0, 3, 4, 7)] == [(0, 0), (0, 3), (1, 0), (1, 3)]


def _worker2d(rank, world, port, cfg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n, k, s, ta, tb, root, pr, pc = cfg
        engines = D.make_grid_engines(lambda g, mem: OracleEngine(g, mem), pr, pc, root)
        A, B, Cin = _inputs(m, n, k, ta, tb, 15)
        i, j = D.grid_coords(rank, pr, pc)
        r0, r1 = D.row_range(m, pr, i)
        n0, n1 = D.row_range(n, pc, j)
        A_loc = np.asfortranarray(A[r0:r1] if ta == "N" else A[:, r0:r1])
        lda = A_loc.shape[0] if A_loc.shape[0] > 0 else 1
        C_loc = np.asfortranarray(Cin[r0:r1, n0:n1]).copy()
        D.dgemm_grid2d(engines, pr, pc, ta, tb, r1 - r0, n, k, 1.5, A_loc, lda,
                       B if rank == root else None, B.shape[0], -0.5, C_loc, max(1, r1 - r0),
                       s, root=root)
        q.put((rank, r0, r1, n0, n1, C_loc))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [
    (37, 50, 40, 9, "N", "N", 0, 2, 2),
    (20, 64, 33, 7, "T", "N", 3, 2, 2),   # root in grid column 1
    (9, 30, 21, 11, "N", "T", 0, 1, 3),   # column blocks only
    (30, 9, 21, 5, "N", "N", 1, 3, 1),    # row blocks only
])
def test_grid2d_broadcast_matches_single_process(cfg):
    m, n, k, s, ta, tb, root, pr, pc = cfg
    parts = _spawn(_worker2d, pr * pc, cfg)
    A, B, Cin = _inputs(m, n, k, ta, tb, 15)
    ref = O.dgemm(ta, tb, m, n, k, 1.5, A, A.shape[0], B, B.shape[0], -0.5, Cin, m, s)
    C = np.full((m, n), np.nan)
    for rank, r0, r1, n0, n1, Cl in parts:
        C[r0:r1, n0:n1] = Cl
    assert np.array_equal(C, ref)
