"""Multi-GPU Ozaki DGEMM: C partitioned into row blocks, B sliced ONCE and its INT8
planes broadcast to every rank (BASELINE north_star).

Rank r owns rows [r0, r1) of C and of op(A) and slices its own A rows (row
exponents are per row -- no communication).  op(B) is sliced on the root only,
chunk by chunk along n; each chunk's B-slice buffer (INT8 planes + int32 column
exponents, ozimmu_b_slices_bytes) goes to all ranks with one NCCL broadcast over
NVLink.  The GEMM on chunk c waits only for chunk c's broadcast, so the transfer
of chunk c+1 overlaps the tensor-core work on chunk c (NCCL's stream vs the
compute stream).  There is no reduction: every C element is computed on exactly
one GPU by the same canonical operation sequence, so C is bitwise identical to the
single-GPU result for every world size.

The math is done by a backend object (``CudaBackend`` wraps the C ABI); the
orchestration here is plain torch.distributed and is unit-tested on CPU with
gloo and a test-only backend.
"""
import torch
import torch.distributed as dist


def row_range(m, world, rank):
    """Balanced contiguous row block [r0, r1) of rank `rank`."""
    return (m * rank) // world, (m * (rank + 1)) // world


def col_chunks(n, chunk_cols):
    chunk_cols = max(1, int(chunk_cols))
    return [(c0, min(n, c0 + chunk_cols)) for c0 in range(0, n, chunk_cols)]


class CudaBackend:
    """Backend over libozimmu (device pointers, column-major, stream = current).

    reserve_sms: SMs kept free of the fused GEMM while broadcasts are in flight.  The GEMM
    is a persistent kernel with one ~227 KB-shared-memory CTA per SM, so an NCCL kernel
    enqueued beside it only runs on SMs it leaves free; without a reserve the broadcast of
    chunk c+1 would wait for the GEMM of chunk c instead of overlapping it.  Pair it with
    NCCL_MAX_CTAS <= reserve_sms (bench.py does)."""

    def __init__(self, handle, device, reserve_sms=0):
        self.h = handle
        self.device = torch.device("cuda", device) if isinstance(device, int) else device
        self.reserve_sms = int(reserve_sms)

    def overlap(self, on):
        """GEMMs leave `reserve_sms` SMs free while `on` (broadcasts in flight)."""
        if self.reserve_sms <= 0:
            return
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        self.h.set_max_sms(max(1, sms - self.reserve_sms) if on else 0)

    def b_slices_bytes(self, n, k, s):
        from .ozimmu import b_slices_bytes
        return b_slices_bytes(n, k, s)

    def alloc(self, nbytes):
        return torch.empty(nbytes, dtype=torch.uint8, device=self.device)

    def bind_stream(self):
        self.h.set_stream(torch.cuda.current_stream(self.device))

    def slice_b(self, transB, k, c0, c1, B, ldb, s, buf):
        # column block [c0, c1) of op(B): N -> columns of B; T/C -> rows of B
        off = c0 * ldb if transB == "N" else c0
        self.h.slice_b(transB, k, c1 - c0, B.data_ptr() + 8 * off, ldb, s, buf)

    def gemm(self, transA, m_loc, c0, c1, k, alpha, A_loc, lda, buf, beta, C_loc, ldc, s):
        self.h.dgemm_presliced_b(transA, m_loc, c1 - c0, k, alpha, A_loc, lda, buf, beta,
                                 C_loc.data_ptr() + 8 * c0 * ldc, ldc, s)


def dgemm_rowblock(backend, transA, transB, m_loc, n, k, alpha, A_loc, lda, B, ldb, beta,
                   C_loc, ldc, s, root=0, chunk_cols=2048, group=None, bufs=None):
    """C_loc = alpha op(A)[r0:r1] op(B) + beta C_loc on every rank.

    A_loc: this rank's rows of op(A) (stored like A, m_loc rows), C_loc its rows of C.
    B is only read on `root` (may be None elsewhere).  Returns the list of per-chunk
    B-slice buffers (reusable via `bufs` to avoid re-allocation)."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    chunks = col_chunks(n, chunk_cols)
    if bufs is None:
        bufs = [backend.alloc(backend.b_slices_bytes(c1 - c0, k, s)) for c0, c1 in chunks]
    works = []
    # root: slice chunk c, then hand it to NCCL (which orders itself after the slicing
    # on the current stream) while slicing chunk c+1
    for (c0, c1), buf in zip(chunks, bufs):
        if rank == root:
            backend.slice_b(transB, k, c0, c1, B, ldb, s, buf)
        if world > 1:
            works.append(dist.broadcast(buf, src=root, group=group, async_op=True))
        else:
            works.append(None)
    overlap = getattr(backend, "overlap", None)
    last = len(chunks) - 1
    for i, ((c0, c1), buf, w) in enumerate(zip(chunks, bufs, works)):
        if w is not None:
            w.wait()  # NCCL: the current stream waits for this chunk only
        if overlap is not None and world > 1:
            overlap(i < last)  # later chunks still in flight: leave SMs to NCCL
        if m_loc > 0:
            backend.gemm(transA, m_loc, c0, c1, k, alpha, A_loc, lda, buf, beta, C_loc, ldc, s)
    if overlap is not None and world > 1:
        overlap(False)
    return bufs


def grid_coords(rank, pr, pc):
    """Rank -> (i, j) on a pr x pc process grid (row-major): C block row i, column block j."""
    return divmod(rank, pc)


def make_grid_groups(pr, pc, root=0):
    """Process groups for dgemm_grid2d: G_j = {root} + the ranks of grid column j.
    Collective: every rank must call it (torch.distributed.new_group), in the same order."""
    groups = []
    for j in range(pc):
        members = sorted({root} | {i * pc + j for i in range(pr)})
        groups.append((members, dist.new_group(ranks=members)))
    return groups


def dgemm_grid2d(backend, transA, transB, m_loc, n, k, alpha, A_loc, lda, B, ldb, beta, C_loc,
                 ldc, s, pr, pc, groups, root=0, chunk_cols=2048, bufs=None):
    """2-D partition of C ('large n'): rank (i, j) of a pr x pc grid owns rows
    row_range(m, pr, i) and columns row_range(n, pc, j) of C.  It slices its own rows of op(A)
    (A row block i is replicated on the pc ranks of grid row i and sliced there, as the survey
    proposes, so there is still no collective but the B one), and receives only the B-slice
    buffers of its column block: the root slices op(B) chunk by chunk and broadcasts chunk c
    of column block j inside group G_j = {root} + column j (make_grid_groups).  Every C element
    is still computed on one GPU by the canonical operation sequence: C is bitwise equal to
    the single-GPU result.  C_loc: this rank's m_loc x n_loc block (ldc); returns the buffers."""
    rank = dist.get_rank()
    i, j = grid_coords(rank, pr, pc)
    plan = []  # (column block jj, c0, c1) in the order the root slices / broadcasts them
    for jj in range(pc):
        n0, n1 = row_range(n, pc, jj)
        for c0, c1 in col_chunks(n1 - n0, chunk_cols):
            plan.append((jj, n0 + c0, n0 + c1))
    mine = [(jj, c0, c1) for jj, c0, c1 in plan if jj == j]
    if bufs is None:
        bufs = {}
    works = {}
    for jj, c0, c1 in plan:
        members, grp = groups[jj]
        if rank not in members:
            continue
        key = (c0, c1)
        if key not in bufs:
            bufs[key] = backend.alloc(backend.b_slices_bytes(c1 - c0, k, s))
        buf = bufs[key]
        if rank == root:
            backend.slice_b(transB, k, c0, c1, B, ldb, s, buf)
        works[key] = dist.broadcast(buf, src=root, group=grp, async_op=True) \
            if len(members) > 1 else None
    n0, _ = row_range(n, pc, j)
    overlap = getattr(backend, "overlap", None)
    for q, (jj, c0, c1) in enumerate(mine):
        w = works.get((c0, c1))
        if w is not None:
            w.wait()
        if overlap is not None:
            overlap(q < len(mine) - 1)
        if m_loc > 0:
            backend.gemm(transA, m_loc, c0 - n0, c1 - n0, k, alpha, A_loc, lda, bufs[(c0, c1)],
                         beta, C_loc, ldc, s)
    if overlap is not None:
        overlap(False)
    # the root may also have broadcast other columns' chunks: complete them before returning
    for key, w in works.items():
        if w is not None and not any((c0, c1) == key for _, c0, c1 in mine):
            w.wait()
    return bufs
