"""Thin ctypes binding over libozimmu.so (include/ozimmu.h).

Argument marshalling only: every step of the method runs in the library's
sm_100a kernels.  PyTorch is used for device memory and streams.  There is no
CPU fallback: if the CUDA library cannot be loaded, or a call fails, an
exception is raised.

The raw entry points keep the C names and BLAS argument order (column-major,
device pointers as ints, alpha/beta as Python floats).  ``matmul`` is the
row-major torch convenience (C = A @ B via C^T = B^T A^T, bitwise identical).
"""
import ctypes as ct
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# OZIMMU_LIB: development override (a variants/ build of the same sources)
LIB_PATH = os.environ.get("OZIMMU_LIB") or os.path.join(HERE, "libozimmu.so")

OP = {"N": 0, "T": 1, "C": 2, 0: 0, 1: 1, 2: 2}
STATUS = {0: "OZIMMU_SUCCESS", 1: "OZIMMU_ERR_INVALID_VALUE", 2: "OZIMMU_ERR_UNSUPPORTED",
          3: "OZIMMU_ERR_WORKSPACE", 4: "OZIMMU_ERR_CUDA", 5: "OZIMMU_ERR_NOT_INITIALIZED",
          6: "OZIMMU_ERR_NCCL"}
NCCL_UNIQUE_ID_BYTES = 128
# int fn(void *ctx, void *buf, size_t bytes, int root, void *stream)  (ozimmu_bcast_fn)
BCAST_FN = ct.CFUNCTYPE(ct.c_int, ct.c_void_p, ct.c_void_p, ct.c_size_t, ct.c_int, ct.c_void_p)
EXP_NONFINITE = 0x7FFFFFFF

# Every symbol include/ozimmu.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "ozimmu_create", "ozimmu_destroy", "ozimmu_set_stream", "ozimmu_workspace_bytes",
    "ozimmu_set_workspace", "ozimmu_get_report", "ozimmu_version", "ozimmu_status_string",
    "ozimmu_dgemm", "ozimmu_b_slices_bytes", "ozimmu_slice_b", "ozimmu_dgemm_presliced_b",
    "ozimmu_debug_split", "ozimmu_debug_level_sums", "ozimmu_debug_pair",
    "ozimmu_timing_enable", "ozimmu_timing_read", "ozimmu_zgemm", "ozimmu_zgemm_workspace_bytes",
    "ozimmu_set_auto", "ozimmu_auto_splits", "ozimmu_dgemm_strided_batched",
    "ozimmu_zgemm_strided_batched", "ozimmu_dgemm_host", "ozimmu_set_max_sms",
    "ozimmu_set_auto_accuracy", "ozimmu_nccl_get_unique_id", "ozimmu_nccl_comm_init",
    "ozimmu_nccl_comm_destroy", "ozimmu_set_dist", "ozimmu_dgemm_nccl", "ozimmu_dgemm_bcast",
    "ozimmu_debug_auto_rho",
]
AUTO_LOSS, AUTO_ACCURACY = 1, 2
AUTO_SMAX_DEFAULT = 18


class OzimmuError(RuntimeError):
    def __init__(self, fn, code):
        super().__init__(f"{fn} failed: {STATUS.get(code, code)}")
        self.code = code


class Timing(ct.Structure):
    _fields_ = [("slice_b_ms", ct.c_float), ("slice_a_ms", ct.c_float), ("gemm_ms", ct.c_float)]


class Report(ct.Structure):
    _fields_ = [("num_slices", ct.c_int), ("slice_width", ct.c_int),
                ("gemm_pairs", ct.c_int64), ("int8_macs", ct.c_int64),
                ("slice_bytes", ct.c_int64), ("tile_n", ct.c_int), ("k_block", ct.c_int),
                ("stages", ct.c_int), ("k_chunks", ct.c_int), ("launches", ct.c_int),
                ("acc_regions", ct.c_int), ("auto_mode", ct.c_int), ("auto_capped", ct.c_int)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def lib():
    """Load libozimmu.so (built in-tree by build.py / __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; "
                           "g.build()'` (no CPU fallback exists)")
    L = ct.CDLL(LIB_PATH)
    i64, i32, vp, dp, sz = ct.c_int64, ct.c_int, ct.c_void_p, ct.POINTER(ct.c_double), ct.c_size_t
    H = ct.c_void_p
    sig = {
        "ozimmu_create": ([ct.POINTER(H), i32], i32),
        "ozimmu_destroy": ([H], i32),
        "ozimmu_set_stream": ([H, vp], i32),
        "ozimmu_set_max_sms": ([H, i32], i32),
        "ozimmu_workspace_bytes": ([i32, i32, i64, i64, i64, i32], sz),
        "ozimmu_set_workspace": ([H, vp, sz], i32),
        "ozimmu_get_report": ([H, ct.POINTER(Report)], i32),
        "ozimmu_version": ([], i32),
        "ozimmu_status_string": ([i32], ct.c_char_p),
        "ozimmu_dgemm": ([H, i32, i32, i64, i64, i64, dp, vp, i64, vp, i64, dp, vp, i64, i32], i32),
        "ozimmu_dgemm_host": ([H, i32, i32, i64, i64, i64, dp, vp, i64, vp, i64, dp, vp, i64, i32],
                              i32),
        "ozimmu_b_slices_bytes": ([i64, i64, i32], sz),
        "ozimmu_slice_b": ([H, i32, i64, i64, vp, i64, i32, vp], i32),
        "ozimmu_dgemm_presliced_b": ([H, i32, i64, i64, i64, dp, vp, i64, vp, dp, vp, i64, i32], i32),
        "ozimmu_debug_split": ([H, i32, i32, i64, i64, vp, i64, i32, vp, vp], i32),
        "ozimmu_debug_auto_rho": ([H, i32, i32, i64, i64, vp, i64, i32, i32, vp], i32),
        "ozimmu_debug_level_sums": ([H, i32, i32, i64, i64, i64, vp, i64, vp, i64, i32, vp], i32),
        "ozimmu_debug_pair": ([H, vp, vp, i64, i64, i64, vp], i32),
        "ozimmu_timing_enable": ([H, i32], i32),
        "ozimmu_zgemm": ([H, i32, i32, i64, i64, i64, dp, vp, i64, vp, i64, dp, vp, i64, i32], i32),
        "ozimmu_zgemm_workspace_bytes": ([i32, i32, i64, i64, i64, i32], sz),
        "ozimmu_set_auto": ([H, ct.c_double, i32], i32),
        "ozimmu_set_auto_accuracy": ([H, ct.c_double, i32], i32),
        "ozimmu_dgemm_strided_batched": ([H, i32, i32, i64, i64, i64, dp, vp, i64, i64, vp, i64,
                                          i64, dp, vp, i64, i64, i64, i32], i32),
        "ozimmu_zgemm_strided_batched": ([H, i32, i32, i64, i64, i64, dp, vp, i64, i64, vp, i64,
                                          i64, dp, vp, i64, i64, i64, i32], i32),
        "ozimmu_auto_splits": ([H, i32, i32, i64, i64, i64, vp, i64, vp, i64, ct.POINTER(i32)], i32),
        "ozimmu_timing_read": ([H, ct.POINTER(Timing), i32], i32),
        "ozimmu_nccl_get_unique_id": ([vp], i32),
        "ozimmu_nccl_comm_init": ([ct.POINTER(vp), i32, vp, i32, i32, i32], i32),
        "ozimmu_nccl_comm_destroy": ([vp], i32),
        "ozimmu_set_dist": ([H, i32, i32, i32], i32),
        "ozimmu_dgemm_nccl": ([H, vp, i32, i32, i32, i64, i64, i64, dp, vp, i64, vp, i64, dp, vp,
                               i64, i32], i32),
        "ozimmu_dgemm_bcast": ([H, BCAST_FN, vp, i32, i32, i32, i32, i32, i64, i64, i64, dp, vp,
                                i64, vp, i64, dp, vp, i64, i32], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(fn, rc):
    if rc != 0:
        raise OzimmuError(fn, rc)


def _d(x):
    return ct.byref(ct.c_double(float(x)))


def _hptr(t):
    """Host address of a CPU torch tensor, a numpy array or an int."""
    if t is None or isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        assert not t.is_cuda, "ozimmu_dgemm_host takes host buffers"
        return t.data_ptr()
    return t.ctypes.data


def _ptr(t):
    """Device pointer of a torch tensor (or an int)."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def workspace_bytes(transA, transB, m, n, k, num_slices):
    return int(lib().ozimmu_workspace_bytes(OP[transA], OP[transB], m, n, k, num_slices))


def b_slices_bytes(n, k, num_slices):
    return int(lib().ozimmu_b_slices_bytes(n, k, num_slices))


def version():
    return int(lib().ozimmu_version())


def nccl_unique_id():
    """128-byte ncclUniqueId from the library's NCCL (call on one rank, share the bytes)."""
    buf = ct.create_string_buffer(NCCL_UNIQUE_ID_BYTES)
    _check("ozimmu_nccl_get_unique_id", lib().ozimmu_nccl_get_unique_id(buf))
    return bytes(buf.raw)


class NcclComm:
    """An NCCL communicator created through libozimmu (ozimmu_nccl_comm_init)."""

    def __init__(self, nranks, uid, rank, device, max_ctas=0):
        assert len(uid) == NCCL_UNIQUE_ID_BYTES
        self.ptr = None
        out = ct.c_void_p()
        idbuf = ct.create_string_buffer(bytes(uid), NCCL_UNIQUE_ID_BYTES)
        _check("ozimmu_nccl_comm_init", lib().ozimmu_nccl_comm_init(
            ct.byref(out), int(nranks), idbuf, int(rank), int(device), int(max_ctas)))
        self.ptr = out.value
        self.rank, self.nranks = rank, nranks

    def close(self):
        if self.ptr:
            lib().ozimmu_nccl_comm_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Handle:
    """Owns an ozimmu handle bound to one CUDA device."""

    def __init__(self, device=0):
        self._h = ct.c_void_p()
        _check("ozimmu_create", lib().ozimmu_create(ct.byref(self._h), int(device)))
        self.device = device
        self._ws = None

    def close(self):
        if self._h:
            lib().ozimmu_destroy(self._h)
            self._h = ct.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing ---------------------------------------------------------------
    def set_stream(self, stream):
        """stream: torch.cuda.Stream, raw cudaStream_t int, or None (legacy default)."""
        raw = None if stream is None else (stream if isinstance(stream, int) else stream.cuda_stream)
        _check("ozimmu_set_stream", lib().ozimmu_set_stream(self._h, raw))

    def set_max_sms(self, max_sms):
        """Cap the SMs of the fused GEMM's persistent grid (0 = all); see ozimmu_set_max_sms."""
        _check("ozimmu_set_max_sms", lib().ozimmu_set_max_sms(self._h, int(max_sms)))

    def set_workspace(self, tensor_or_ptr, nbytes=None):
        if tensor_or_ptr is None:
            self._ws = None
            _check("ozimmu_set_workspace", lib().ozimmu_set_workspace(self._h, None, 0))
            return
        if nbytes is None:
            nbytes = tensor_or_ptr.numel() * tensor_or_ptr.element_size()
        self._ws = tensor_or_ptr  # keep alive
        _check("ozimmu_set_workspace",
               lib().ozimmu_set_workspace(self._h, _ptr(tensor_or_ptr), int(nbytes)))

    def report(self):
        r = Report()
        _check("ozimmu_get_report", lib().ozimmu_get_report(self._h, ct.byref(r)))
        return r.as_dict()

    def timing_enable(self, max_calls):
        _check("ozimmu_timing_enable", lib().ozimmu_timing_enable(self._h, int(max_calls)))

    def timing_read(self, max_out=4096):
        buf = (Timing * max_out)()
        n = lib().ozimmu_timing_read(self._h, buf, max_out)
        if n < 0:
            raise OzimmuError("ozimmu_timing_read", 4)
        return [{"slice_b_ms": buf[i].slice_b_ms, "slice_a_ms": buf[i].slice_a_ms,
                 "gemm_ms": buf[i].gemm_ms} for i in range(min(n, max_out))]

    # -- the C ABI, same names and argument order ---------------------------------
    def dgemm(self, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, num_slices):
        _check("ozimmu_dgemm", lib().ozimmu_dgemm(
            self._h, OP[transA], OP[transB], m, n, k, _d(alpha), _ptr(A), lda, _ptr(B), ldb,
            _d(beta), _ptr(C), ldc, int(num_slices)))

    def dgemm_host(self, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc,
                   num_slices):
        """ozimmu_dgemm with A, B, C in host memory (CPU torch tensors, pinned for overlap,
        or numpy arrays / raw addresses); blocks until C is written."""
        _check("ozimmu_dgemm_host", lib().ozimmu_dgemm_host(
            self._h, OP[transA], OP[transB], m, n, k, _d(alpha), _hptr(A), lda, _hptr(B), ldb,
            _d(beta), _hptr(C), ldc, int(num_slices)))

    def set_auto(self, threshold, s_max=AUTO_SMAX_DEFAULT):
        """INT8-AUTO with the paper's mean-mantissa-loss rule (reading A17) for
        num_slices = 0 calls."""
        _check("ozimmu_set_auto", lib().ozimmu_set_auto(self._h, float(threshold), int(s_max)))

    def set_auto_accuracy(self, tau=1.0, s_max=AUTO_SMAX_DEFAULT):
        """INT8-AUTO with the k-aware accuracy-targeted rule (reading A18, the default):
        predicted error <= tau x FP64 DGEMM's probabilistic error level."""
        _check("ozimmu_set_auto_accuracy",
               lib().ozimmu_set_auto_accuracy(self._h, float(tau), int(s_max)))

    def auto_splits(self, transA, transB, m, n, k, A, lda, B, ldb):
        out = ct.c_int()
        _check("ozimmu_auto_splits", lib().ozimmu_auto_splits(
            self._h, OP[transA], OP[transB], m, n, k, _ptr(A), lda, _ptr(B), ldb, ct.byref(out)))
        return out.value

    def zgemm(self, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, num_slices):
        """Complex GEMM: A, B, C interleaved complex (e.g. torch.complex128), ld in complex
        elements, alpha / beta Python complex numbers."""
        a = (ct.c_double * 2)(complex(alpha).real, complex(alpha).imag)
        b = (ct.c_double * 2)(complex(beta).real, complex(beta).imag)
        _check("ozimmu_zgemm", lib().ozimmu_zgemm(
            self._h, OP[transA], OP[transB], m, n, k, a, _ptr(A), lda, _ptr(B), ldb, b, _ptr(C),
            ldc, int(num_slices)))

    def dgemm_strided_batched(self, transA, transB, m, n, k, alpha, A, lda, strideA, B, ldb,
                              strideB, beta, C, ldc, strideC, batch, num_slices):
        _check("ozimmu_dgemm_strided_batched", lib().ozimmu_dgemm_strided_batched(
            self._h, OP[transA], OP[transB], m, n, k, _d(alpha), _ptr(A), lda, strideA, _ptr(B),
            ldb, strideB, _d(beta), _ptr(C), ldc, strideC, batch, int(num_slices)))

    def zgemm_strided_batched(self, transA, transB, m, n, k, alpha, A, lda, strideA, B, ldb,
                              strideB, beta, C, ldc, strideC, batch, num_slices):
        a = (ct.c_double * 2)(complex(alpha).real, complex(alpha).imag)
        b = (ct.c_double * 2)(complex(beta).real, complex(beta).imag)
        _check("ozimmu_zgemm_strided_batched", lib().ozimmu_zgemm_strided_batched(
            self._h, OP[transA], OP[transB], m, n, k, a, _ptr(A), lda, strideA, _ptr(B), ldb,
            strideB, b, _ptr(C), ldc, strideC, batch, int(num_slices)))

    def slice_b(self, transB, k, n, B, ldb, num_slices, b_slices):
        _check("ozimmu_slice_b", lib().ozimmu_slice_b(
            self._h, OP[transB], k, n, _ptr(B), ldb, int(num_slices), _ptr(b_slices)))

    def dgemm_presliced_b(self, transA, m, n, k, alpha, A, lda, b_slices, beta, C, ldc,
                          num_slices):
        _check("ozimmu_dgemm_presliced_b", lib().ozimmu_dgemm_presliced_b(
            self._h, OP[transA], m, n, k, _d(alpha), _ptr(A), lda, _ptr(b_slices), _d(beta),
            _ptr(C), ldc, int(num_slices)))

    def debug_split(self, op, is_rows, rows, kdim, M, ld, num_slices, planes_out, exps_out):
        _check("ozimmu_debug_split", lib().ozimmu_debug_split(
            self._h, OP[op], int(is_rows), rows, kdim, _ptr(M), ld, int(num_slices),
            _ptr(planes_out), _ptr(exps_out)))

    def debug_auto_rho(self, op, is_rows, rows, kdim, M, ld, w, s_max):
        """Device statistics of the accuracy AUTO rule for one operand: rho[0..s_max] (numpy)."""
        out = (ct.c_double * (s_max + 1))()
        _check("ozimmu_debug_auto_rho", lib().ozimmu_debug_auto_rho(
            self._h, OP[op], int(is_rows), rows, kdim, _ptr(M), ld, int(w), int(s_max), out))
        import numpy as _np
        return _np.array(out[:], dtype=_np.float64)

    def debug_level_sums(self, transA, transB, m, n, k, A, lda, B, ldb, num_slices, Lg_out):
        _check("ozimmu_debug_level_sums", lib().ozimmu_debug_level_sums(
            self._h, OP[transA], OP[transB], m, n, k, _ptr(A), lda, _ptr(B), ldb,
            int(num_slices), _ptr(Lg_out)))

    def debug_pair(self, Ai, Bj, m, n, k, P_out):
        _check("ozimmu_debug_pair", lib().ozimmu_debug_pair(
            self._h, _ptr(Ai), _ptr(Bj), m, n, k, _ptr(P_out)))

    # -- multi-GPU (include/ozimmu.h "multi-GPU") ----------------------------
    def set_dist(self, chunk_cols=0, reserve_sms=8, bcast_fp64=False):
        _check("ozimmu_set_dist", lib().ozimmu_set_dist(self._h, int(chunk_cols),
                                                        int(reserve_sms), int(bool(bcast_fp64))))

    def dgemm_nccl(self, comm, root, transA, transB, m_local, n, k, alpha, A_local, lda, B, ldb,
                   beta, C_local, ldc, num_slices):
        """C row blocks over an NCCL communicator (comm: NcclComm or raw ncclComm_t int)."""
        raw = comm if isinstance(comm, int) else comm.ptr
        _check("ozimmu_dgemm_nccl", lib().ozimmu_dgemm_nccl(
            self._h, raw, int(root), OP[transA], OP[transB], m_local, n, k, _d(alpha),
            _ptr(A_local), lda, _ptr(B), ldb, _d(beta), _ptr(C_local), ldc, int(num_slices)))

    def dgemm_bcast(self, fn, rank, nranks, root, transA, transB, m_local, n, k, alpha, A_local,
                    lda, B, ldb, beta, C_local, ldc, num_slices):
        """The same driver over a caller broadcast fn (a BCAST_FN; keep it alive)."""
        _check("ozimmu_dgemm_bcast", lib().ozimmu_dgemm_bcast(
            self._h, fn, None, int(rank), int(nranks), int(root), OP[transA], OP[transB], m_local,
            n, k, _d(alpha), _ptr(A_local), lda, _ptr(B), ldb, _d(beta), _ptr(C_local), ldc,
            int(num_slices)))

    # -- torch convenience --------------------------------------------------------
    def matmul(self, A, B, num_slices, out=None):
        """Row-major torch float64 CUDA tensors: returns A @ B (m x n) computed by the
        Ozaki scheme.  Uses C^T = B^T A^T on the column-major ABI."""
        import torch
        assert A.is_cuda and B.is_cuda and A.dtype == torch.float64 and B.dtype == torch.float64
        A = A.contiguous()
        B = B.contiguous()
        m, k = A.shape
        k2, n = B.shape
        assert k == k2
        if out is None:
            out = torch.empty((m, n), dtype=torch.float64, device=A.device)
        self.dgemm("N", "N", n, m, k, 1.0, B, n, A, k, 0.0, out, n, num_slices)
        return out
