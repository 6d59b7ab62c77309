"""World-size-2 run of the multi-GPU driver (paper_2306_11975_b200/dist.py) with the real CUDA
backend: two processes share cuda:0 (the test box has one GPU), torch.distributed over gloo
(NCCL refuses two ranks on one device).  Root slices op(B) chunk by chunk with
ozimmu_slice_b, the B-slice buffers are broadcast, each rank runs
ozimmu_dgemm_presliced_b on its row block; the assembled C must equal the single-call
ozimmu_dgemm result bit for bit and the CPU oracle (C row blocks, one broadcast
of B's INT8 planes, no reduction)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(cfg):
    m, n, k, s, ta, tb, root, chunk = cfg
    A = synth.gen_phi(*((m, k) if ta == "N" else (k, m)), 0.5, 11)
    B = synth.gen_phi(*((k, n) if tb == "N" else (n, k)), 0.5, 12)
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
        dev = torch.device("cuda", 0)
        m, n, k, s, ta, tb, root, chunk = cfg
        A, B, Cin = _inputs(cfg)
        r0, r1 = D.row_range(m, world, rank)
        ml = r1 - r0
        A_loc = np.asfortranarray(A[r0:r1] if ta == "N" else A[:, r0:r1])
        lda = max(1, A_loc.shape[0])
        dA = torch.from_numpy(A_loc.ravel(order="F").copy()).to(dev)
        dB = torch.from_numpy(B.ravel(order="F").copy()).to(dev) if rank == root else None
        C_loc = np.asfortranarray(Cin[r0:r1])
        dC = torch.from_numpy(C_loc.ravel(order="F").copy()).to(dev)
        h = oz.Handle(0)
        h.set_stream(torch.cuda.current_stream(dev))
        be = D.CudaBackend(h, dev, reserve_sms=21)  # capped GEMM grid (127 SMs) while in flight
        D.dgemm_rowblock(be, ta, tb, ml, n, k, 1.5, dA, lda, dB, B.shape[0], -0.5,
                         dC, max(1, ml), s, root=root, chunk_cols=chunk)
        torch.cuda.synchronize()
        q.put((rank, r0, r1, dC.cpu().numpy().reshape(n, ml).T.copy() if ml else None))
        h.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [
    (300, 200, 130, 9, "N", "N", 0, 64),
    (257, 96, 1000, 7, "T", "N", 1, 48),
    (64, 150, 77, 13, "N", "T", 0, 100),
])
def test_rowblock_broadcast_cuda_backend_bitwise(cfg):
    import oracle as O
    import paper_2306_11975_b200 as oz
    world = 2
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
    m, n, k, s, ta, tb, root, chunk = cfg
    A, B, Cin = _inputs(cfg)
    C = np.zeros((m, n))
    for rank, r0, r1, Cl in parts:
        if Cl is not None:
            C[r0:r1] = Cl
    # single-call reference on the GPU
    dev = torch.device("cuda", 0)
    h = oz.Handle(0)
    dA = torch.from_numpy(A.ravel(order="F").copy()).to(dev)
    dB = torch.from_numpy(B.ravel(order="F").copy()).to(dev)
    dC = torch.from_numpy(Cin.ravel(order="F").copy()).to(dev)
    h.dgemm(ta, tb, m, n, k, 1.5, dA, A.shape[0], dB, B.shape[0], -0.5, dC, m, s)
    torch.cuda.synchronize()
    one = dC.cpu().numpy().reshape(n, m).T
    h.close()
    assert np.array_equal(C, one)
    ref = O.dgemm(ta, tb, m, n, k, 1.5, A, A.shape[0], B, B.shape[0], -0.5, Cin, m, s)
    assert np.array_equal(C, ref)


def _worker2d(rank, world, port, cfg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import paper_2306_11975_b200 as oz
    from paper_2306_11975_b200 import dist as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        m, n, k, s, ta, tb, root, chunk, pr, pc = cfg
        groups = D.make_grid_groups(pr, pc, root)
        A, B, Cin = _inputs(cfg[:8])
        i, j = D.grid_coords(rank, pr, pc)
        r0, r1 = D.row_range(m, pr, i)
        n0, n1 = D.row_range(n, pc, j)
        ml = r1 - r0
        A_loc = np.asfortranarray(A[r0:r1] if ta == "N" else A[:, r0:r1])
        dA = torch.from_numpy(A_loc.ravel(order="F").copy()).to(dev)
        dB = torch.from_numpy(B.ravel(order="F").copy()).to(dev) if rank == root else None
        dC = torch.from_numpy(np.asfortranarray(Cin[r0:r1, n0:n1]).ravel(order="F").copy()).to(dev)
        h = oz.Handle(0)
        h.set_stream(torch.cuda.current_stream(dev))
        be = D.CudaBackend(h, dev, reserve_sms=16)
        D.dgemm_grid2d(be, ta, tb, ml, n, k, 1.5, dA, max(1, A_loc.shape[0]), dB, B.shape[0],
                       -0.5, dC, max(1, ml), s, pr, pc, groups, root=root, chunk_cols=chunk)
        torch.cuda.synchronize()
        q.put((rank, r0, r1, n0, n1, dC.cpu().numpy().reshape(n1 - n0, ml).T.copy()))
        h.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [(300, 260, 130, 9, "N", "N", 0, 64, 2, 2),
                                 (200, 150, 500, 13, "T", "T", 3, 48, 2, 2)])
def test_grid2d_cuda_backend_bitwise(cfg):
    import oracle as O
    m, n, k, s, ta, tb, root, chunk, pr, pc = cfg
    world = pr * pc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker2d, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    A, B, Cin = _inputs(cfg[:8])
    C = np.full((m, n), np.nan)
    for rank, r0, r1, n0, n1, Cl in parts:
        C[r0:r1, n0:n1] = Cl
    ref = O.dgemm(ta, tb, m, n, k, 1.5, A, A.shape[0], B, B.shape[0], -0.5, Cin, m, s)
    assert np.array_equal(C, ref)
