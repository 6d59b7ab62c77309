"""Multi-GPU Ozaki DGEMM: thin orchestration over the library's multi-GPU driver (
BASELINE north_star: C in row blocks, 2-D blocks for large n; every GPU slices its own A rows;
B's slices are computed once and NCCL-broadcast over NVLink; no other collective).

The data path -- chunked slicing of op(B) on the root, the NCCL broadcasts on the handle's
collective stream, the per-chunk GEMMs that wait only for their chunk, the SM reservation while
broadcasts are in flight -- is inside libozimmu (csrc/dist.cu, ``ozimmu_dgemm_nccl``).  This
module only decides who owns which rows / columns, creates the communicators (the NCCL unique
id travels over torch.distributed, any backend), and makes the calls in a deadlock-free order.

Engines (``engine.dgemm(root, transA, transB, m_loc, n, k, alpha, A_loc, lda, B, ldb, beta,
C_loc, ldc, s)``, one call per rank of the engine's group):
  * ``NcclEngine``  -- the product: ozimmu_dgemm_nccl over an NCCL communicator.
  * ``BcastEngine`` -- the same library driver over a host-staged torch.distributed broadcast
    (ozimmu_dgemm_bcast): runs the multi-rank logic where NCCL cannot (several ranks on one
    GPU, gloo); used by the tests.
The CPU tests plug in an oracle-backed engine to check the partitioning logic here.
"""

import torch
import torch.distributed as dist


def row_range(m, world, rank):
    """Balanced contiguous block [r0, r1) of rank `rank` out of `world`."""
    return (m * rank) // world, (m * (rank + 1)) // world


def grid_coords(rank, pr, pc):
    """Rank -> (i, j) on a pr x pc process grid (row-major): C block row i, column block j."""
    return divmod(rank, pc)


def grid_members(pr, pc, root, j):
    """Ranks of the broadcast group of grid column j: the root plus the ranks of column j."""
    return sorted({root} | {i * pc + j for i in range(pr)})


# ---- engines ---------------------------------------------------------------------------

def make_nccl_comm(device, group=None, max_ctas=0, members=None):
    """An NCCL communicator over `group` (all ranks if None) created by libozimmu; the unique
    id goes from the group's first member to the others over torch.distributed.  Collective
    over the group.  max_ctas caps the communicator's CTAs (pair with the handle's
    reserve_sms)."""
    from .ozimmu import NcclComm, nccl_unique_id
    if members is None:
        members = list(range(dist.get_world_size()))
    rank = dist.get_rank()
    src = members[0]
    obj = [nccl_unique_id() if rank == src else None]
    if len(members) > 1:
        dist.broadcast_object_list(obj, src=src, group=group)
    return NcclComm(len(members), obj[0], members.index(rank), device, max_ctas)


class NcclEngine:
    """ozimmu_dgemm_nccl on `handle` over `comm` (an NcclComm); `root` is a rank of the comm."""

    def __init__(self, handle, comm):
        self.h, self.comm = handle, comm
        self.launches = 0  # kernels the library launched for the last call

    def dgemm(self, root, transA, transB, m_loc, n, k, alpha, A_loc, lda, B, ldb, beta, C_loc,
              ldc, s):
        self.h.dgemm_nccl(self.comm, root, transA, transB, m_loc, n, k, alpha, A_loc, lda, B,
                          ldb, beta, C_loc, ldc, s)
        self.launches = self.h.report()["launches"]


class BcastEngine:
    """ozimmu_dgemm_bcast on `handle` with a synchronous host-staged broadcast over the
    torch.distributed `group` (members: its global ranks in group order; `root` is an index
    into them).  The callback synchronises the library's collective stream, copies the device
    bytes to the host, broadcasts them and copies them back before returning, which satisfies
    the ozimmu_bcast_fn ordering contract."""

    def __init__(self, handle, group=None, members=None):
        from .ozimmu import BCAST_FN
        self.h, self.group = handle, group
        self.members = members if members is not None else list(range(dist.get_world_size()))
        self.me = self.members.index(dist.get_rank())
        self.calls = 0
        self.launches = 0  # kernels the library launched for the last call
        self._fn = BCAST_FN(self._bcast)  # kept alive with the engine

    def _bcast(self, ctx, buf, nbytes, root, stream):
        try:
            from cuda.bindings import runtime as rt
            rt.cudaStreamSynchronize(stream)
            host = torch.empty(int(nbytes), dtype=torch.uint8)
            if self.me == root:
                rt.cudaMemcpy(host.data_ptr(), buf, int(nbytes),
                              rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
            if len(self.members) > 1:
                dist.broadcast(host, src=self.members[root], group=self.group)
            if self.me != root:
                rt.cudaMemcpy(buf, host.data_ptr(), int(nbytes),
                              rt.cudaMemcpyKind.cudaMemcpyHostToDevice)
            self.calls += 1
            return 0
        except Exception:  # reported to the library as a failed broadcast (OZIMMU_ERR_NCCL)
            return 1

    def dgemm(self, root, transA, transB, m_loc, n, k, alpha, A_loc, lda, B, ldb, beta, C_loc,
              ldc, s):
        self.h.dgemm_bcast(self._fn, self.me, len(self.members), root, transA, transB, m_loc, n,
                           k, alpha, A_loc, lda, B, ldb, beta, C_loc, ldc, s)
        self.launches = self.h.report()["launches"]


# ---- partitions ------------------------------------------------------------------------

def dgemm_rowblock(engine, transA, transB, m_loc, n, k, alpha, A_loc, lda, B, ldb, beta, C_loc,
                   ldc, s, root=0):
    """C_loc = alpha op(A)[r0:r1] op(B) + beta C_loc on every rank (row_range gives [r0, r1)).

    A_loc: this rank's rows of op(A) (stored like A, m_loc rows); C_loc: its rows of C.  B is
    only read on `root` (may be None elsewhere); ldb must be the same on every rank."""
    engine.dgemm(root, transA, transB, m_loc, n, k, alpha, A_loc, lda, B, ldb, beta, C_loc, ldc,
                 s)


def _col_block(transB, B, ldb, n0):
    """Column n0 onwards of op(B): a device pointer (int) for torch tensors / ints, a view for
    numpy arrays (the CPU test engine), None on non-root ranks."""
    if B is None:
        return None
    if hasattr(B, "__array_interface__"):
        return B[:, n0:] if transB == "N" else B[n0:, :]
    base = B if isinstance(B, int) else B.data_ptr()
    return base + 8 * (n0 * ldb if transB == "N" else n0)


def dgemm_grid2d(engines, pr, pc, transA, transB, m_loc, n, k, alpha, A_loc, lda, B, ldb, beta,
                 C_loc, ldc, s, root=0):
    """2-D partition of C ('large n'): rank (i, j) of a pr x pc grid owns rows
    row_range(m, pr, i) and columns row_range(n, pc, j) of C.  It slices its own rows of op(A)
    (row block i is replicated on the pc ranks of grid row i, so the B broadcast stays the only
    collective) and receives only the B slices of column block j, broadcast by the root inside
    G_j = grid_members(pr, pc, root, j).  engines[j]: the engine of G_j on this rank (None if
    the rank is not in G_j).  Every rank walks j = 0 .. pc-1 in the same order; the root takes
    part in every G_j (m_loc = 0 where it owns no block).  C_loc: this rank's m_loc x n_loc
    block (ldc)."""
    rank = dist.get_rank()
    i, j = grid_coords(rank, pr, pc)
    for jj in range(pc):
        eng = engines[jj]
        if eng is None:
            continue
        n0, n1 = row_range(n, pc, jj)
        mine = jj == j
        members = grid_members(pr, pc, root, jj)
        eng.dgemm(members.index(root), transA, transB, m_loc if mine else 0, n1 - n0, k, alpha,
                  A_loc if mine else None, lda, _col_block(transB, B, ldb, n0) if rank == root
                  else None, ldb, beta, C_loc if mine else None, ldc, s)


def make_grid_engines(make_engine, pr, pc, root=0):
    """engines[j] for dgemm_grid2d: make_engine(group, members) for every G_j this rank is in.
    Collective: every rank must call it (torch.distributed.new_group), in the same order."""
    rank = dist.get_rank()
    out = []
    for jj in range(pc):
        members = grid_members(pr, pc, root, jj)
        grp = dist.new_group(ranks=members)
        out.append(make_engine(grp, members) if rank in members else None)
    return out
