"""ctypes wrapper over oracle/liboracle.so (ozaki_ref.c + dd_ref.c).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Arrays follow the BLAS
column-major convention: a matrix buffer is a numpy float64 array (any shape,
Fortran/contiguous memory) addressed as ``M[i + j*ld]``.
"""
import ctypes as ct
import os

import numpy as np

from . import build as _build

_lib = None

OP = {"N": 0, "T": 1, "C": 2, 0: 0, 1: 1, 2: 2}


def lib():
    global _lib
    if _lib is None:
        path = _build.build()
        L = ct.CDLL(path)
        i64, i32, dbl, vp = ct.c_int64, ct.c_int, ct.c_double, ct.c_void_p
        L.oz_ref_alpha.argtypes = [i32, i64]
        L.oz_ref_alpha.restype = i32
        L.oz_ref_bps.argtypes = [i32, i32, i64]
        L.oz_ref_bps.restype = i32
        L.oz_ref_slice_width.argtypes = [i64]
        L.oz_ref_slice_width.restype = i32
        L.oz_ref_budget_ok.argtypes = [i32, i64]
        L.oz_ref_budget_ok.restype = i32
        L.oz_ref_gemm_count.argtypes = [i32]
        L.oz_ref_gemm_count.restype = i64
        L.oz_ref_split.argtypes = [i32, i64, i64, vp, i64, i32, i32, vp, vp, vp]
        L.oz_ref_split.restype = i32
        L.oz_ref_int_gemm.argtypes = [i64, i64, i64, vp, vp, vp]
        L.oz_ref_int_gemm.restype = i32
        L.oz_ref_dgemm_sub.argtypes = [i32, i32, i64, i64, i64, dbl, vp, i64, vp, i64, dbl, vp,
                                       i64, i32, i32, vp, i64, vp, i64]
        L.oz_ref_dgemm_sub.restype = i32
        L.oz_ref_level_sums_sub.argtypes = [i32, i32, i64, i64, i64, vp, i64, vp, i64, i32,
                                            vp, i64, vp, i64, vp]
        L.oz_ref_level_sums_sub.restype = i32
        L.oz_ref_zgemm_sub.argtypes = [i32, i32, i64, i64, i64, vp, vp, i64, vp, i64, vp, vp,
                                       i64, i32, vp, i64, vp, i64]
        L.oz_ref_zgemm_sub.restype = i32
        L.dd_zgemm_sub.argtypes = [i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64,
                                   vp, vp, vp, vp]
        L.dd_zgemm_sub.restype = i32
        L.oz_ref_mantissa_loss.argtypes = [i32, i64, i64, vp, i64, i32, i32, vp, vp]
        L.oz_ref_mantissa_loss.restype = i32
        L.oz_ref_auto_splits.argtypes = [i32, i32, i64, i64, i64, vp, i64, vp, i64, dbl, i32]
        L.oz_ref_auto_splits.restype = i32
        L.oz_ref_trunc_residual.argtypes = [i32, i64, i64, vp, i64, i32, i32, vp]
        L.oz_ref_trunc_residual.restype = i32
        L.oz_ref_acc_eta.argtypes = [vp, vp, i32]
        L.oz_ref_acc_eta.restype = dbl
        L.oz_ref_auto_splits_acc.argtypes = [i32, i32, i64, i64, i64, vp, i64, vp, i64, dbl, i32,
                                             ct.POINTER(i32)]
        L.oz_ref_auto_splits_acc.restype = i32
        L.dd_two_sum.argtypes = [dbl, dbl, ct.POINTER(dbl), ct.POINTER(dbl)]
        L.dd_two_prod.argtypes = [dbl, dbl, ct.POINTER(dbl), ct.POINTER(dbl)]
        L.dd_gemm_sub.argtypes = [i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64,
                                  vp, vp]
        L.dd_gemm_sub.restype = i32
        L.fp64_gemm_sub.argtypes = [i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64,
                                    vp]
        L.fp64_gemm_sub.restype = i32
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ct.c_void_p) if a is not None else None


def _f64(a):
    a = np.asarray(a, dtype=np.float64)
    # keep memory order as given (column-major buffers are usually Fortran arrays)
    if not (a.flags.f_contiguous or a.flags.c_contiguous):
        a = np.asfortranarray(a)
    return a


def _idx(v, n):
    if v is None:
        return np.arange(n, dtype=np.int64)
    return np.ascontiguousarray(np.asarray(v, dtype=np.int64))


# --- A1 planner -------------------------------------------------------------

def alpha(l_acc, k):
    return lib().oz_ref_alpha(int(l_acc), int(k))


def bps(l_in, l_acc, k):
    return lib().oz_ref_bps(int(l_in), int(l_acc), int(k))


def slice_width(k):
    return lib().oz_ref_slice_width(int(k))


def budget_ok(w, k):
    return bool(lib().oz_ref_budget_ok(int(w), int(k)))


def gemm_count(s):
    return int(lib().oz_ref_gemm_count(int(s)))


# --- A2/A3 split -------------------------------------------------------------

def split(M, trans, rows, kdim, ld, s, w):
    """Split `rows` vectors of length `kdim`: v(r,l) = M[r + l*ld] (trans 0) or
    M[l + r*ld] (trans 1).  Returns (digits[s][rows][kdim] int8, E int32, nonfinite uint8)."""
    M = _f64(M)
    d = np.zeros((s, rows, kdim), dtype=np.int8)
    E = np.zeros(rows, dtype=np.int32)
    bad = np.zeros(rows, dtype=np.uint8)
    rc = lib().oz_ref_split(int(trans), rows, kdim, _p(M), int(ld), int(s), int(w), _p(d), _p(E),
                            _p(bad))
    if rc:
        raise ValueError(f"oz_ref_split failed rc={rc}")
    return d, E, bad


def split_opA(A, transA, m, k, lda, s, w=None):
    """Rows of op(A) (m x k)."""
    w = slice_width(k) if w is None else w
    return split(A, 0 if OP[transA] == 0 else 1, m, k, lda, s, w)


def split_opB(B, transB, k, n, ldb, s, w=None):
    """Columns of op(B) (k x n), returned as digits[s][n][k]."""
    w = slice_width(k) if w is None else w
    return split(B, 1 if OP[transB] == 0 else 0, n, k, ldb, s, w)


# --- A4 -------------------------------------------------------------------------

def int_gemm(a, b):
    """a: [ra][k] int8, b: [rb][k] int8 (columns of op(B)) -> [ra][rb] int32."""
    a = np.ascontiguousarray(a, dtype=np.int8)
    b = np.ascontiguousarray(b, dtype=np.int8)
    ra, k = a.shape
    rb, k2 = b.shape
    assert k == k2
    P = np.zeros((ra, rb), dtype=np.int32)
    rc = lib().oz_ref_int_gemm(ra, rb, k, _p(a), _p(b), _p(P))
    if rc:
        raise OverflowError("INT32 partial sum overflow")
    return P


# --- A5 full method -------------------------------------------------------------

def dgemm(transA, transB, m, n, k, alpha_, A, lda, B, ldb, beta, C, ldc, s, mode="L",
          rows=None, cols=None):
    """Ozaki-scheme DGEMM.  Returns a copy of C (same buffer layout) with the
    selected rows x cols block overwritten.  mode 'L' = canonical level order
    (parity target), 'P' = paper-literal Alg. 3 order."""
    A = _f64(A)
    B = _f64(B)
    Cout = np.array(C, dtype=np.float64, copy=True, order="K")
    ri, cj = _idx(rows, m), _idx(cols, n)
    rc = lib().oz_ref_dgemm_sub(OP[transA], OP[transB], m, n, k, float(alpha_), _p(A), lda,
                                _p(B), ldb, float(beta), _p(Cout), ldc, int(s),
                                0 if mode == "L" else 1, _p(ri), len(ri), _p(cj), len(cj))
    if rc:
        raise ValueError(f"oz_ref_dgemm_sub failed rc={rc}")
    return Cout


def dgemm_simple(A, B, s, mode="L", alpha_=1.0, beta=0.0, C=None, transA="N", transB="N",
                 rows=None, cols=None):
    """Convenience: A, B numpy 2-D arrays holding the *stored* matrices
    (column-major semantics via Fortran order)."""
    A = np.asfortranarray(A, dtype=np.float64)
    B = np.asfortranarray(B, dtype=np.float64)
    m = A.shape[0] if OP[transA] == 0 else A.shape[1]
    k = A.shape[1] if OP[transA] == 0 else A.shape[0]
    n = B.shape[1] if OP[transB] == 0 else B.shape[0]
    if C is None:
        C = np.zeros((m, n), dtype=np.float64, order="F")
    C = np.asfortranarray(C, dtype=np.float64)
    return dgemm(transA, transB, m, n, k, alpha_, A, A.shape[0], B, B.shape[0], beta, C, m, s,
                 mode, rows, cols)


def level_sums(transA, transB, m, n, k, A, lda, B, ldb, s, rows=None, cols=None):
    """Exact level sums L_g (g = 2..s+1) -> int64 [s][nr][nc]."""
    A = _f64(A)
    B = _f64(B)
    ri, cj = _idx(rows, m), _idx(cols, n)
    out = np.zeros((s, len(ri), len(cj)), dtype=np.int64)
    rc = lib().oz_ref_level_sums_sub(OP[transA], OP[transB], m, n, k, _p(A), lda, _p(B), ldb,
                                     int(s), _p(ri), len(ri), _p(cj), len(cj), _p(out))
    if rc:
        raise ValueError(f"oz_ref_level_sums_sub failed rc={rc}")
    return out


def mantissa_loss(M, trans, rows, kdim, ld, w, s_max):
    """f2 (reading A17): (loss_sum[s-1] for s = 1..s_max, nnz) over the vectors of op(M)."""
    M = _f64(M)
    ls = np.zeros(s_max, dtype=np.int64)
    nnz = np.zeros(1, dtype=np.int64)
    rc = lib().oz_ref_mantissa_loss(int(trans), rows, kdim, _p(M), int(ld), int(w), int(s_max),
                                    _p(ls), _p(nnz))
    if rc:
        raise ValueError("oz_ref_mantissa_loss failed")
    return ls, int(nnz[0])


def auto_splits(transA, transB, m, n, k, A, lda, B, ldb, T, s_max=32):
    """f2 INT8-AUTO: smallest s with both mean mantissa losses <= T."""
    A = _f64(A)
    B = _f64(B)
    s = lib().oz_ref_auto_splits(OP[transA], OP[transB], m, n, k, _p(A), lda, _p(B), ldb,
                                 float(T), int(s_max))
    if s < 0:
        raise ValueError("oz_ref_auto_splits failed")
    return s


def trunc_residual(M, trans, rows, kdim, ld, w, s_max):
    """f2 accuracy-targeted AUTO (reading A18): rho[t], t = 0..s_max = max over the vectors
    of op(M) of the relative l1 truncation residual after t digits (fixed-point, upper
    estimate).  trans 0: vector r = M[r + l*ld]; 1: M[l + r*ld]."""
    M = _f64(M)
    rho = np.zeros(s_max + 1)
    rc = lib().oz_ref_trunc_residual(int(trans), rows, kdim, _p(M), int(ld), int(w), int(s_max),
                                     _p(rho))
    if rc:
        raise ValueError(f"oz_ref_trunc_residual failed rc={rc}")
    return rho


def acc_eta(rhoA, rhoB, s):
    """eta(s) = sum_{t=0..s} rhoA[t] rhoB[s-t] (reading A18)."""
    ra = np.ascontiguousarray(rhoA, dtype=np.float64)
    rb = np.ascontiguousarray(rhoB, dtype=np.float64)
    return lib().oz_ref_acc_eta(_p(ra), _p(rb), int(s))


def auto_splits_acc(transA, transB, m, n, k, A, lda, B, ldb, tau=1.0, s_max=18):
    """f2 accuracy-targeted INT8-AUTO (reading A18): (s, capped)."""
    A = _f64(A)
    B = _f64(B)
    capped = ct.c_int(0)
    s = lib().oz_ref_auto_splits_acc(OP[transA], OP[transB], m, n, k, _p(A), lda, _p(B), ldb,
                                     float(tau), int(s_max), ct.byref(capped))
    if s < 0:
        raise ValueError("oz_ref_auto_splits_acc failed")
    return s, bool(capped.value)


def _c128(a):
    a = np.asarray(a, dtype=np.complex128)
    if not (a.flags.f_contiguous or a.flags.c_contiguous):
        a = np.asfortranarray(a)
    return a


def zgemm(transA, transB, m, n, k, alpha_, A, lda, B, ldb, beta, C, ldc, s, rows=None,
          cols=None):
    """Complex Ozaki GEMM (reading A16: real embedding with interleaved K, mode L).
    A, B, C: complex128 buffers addressed column-major (X[i + j*ld]).  Returns a copy of C."""
    A = _c128(A)
    B = _c128(B)
    Cout = np.array(C, dtype=np.complex128, copy=True, order="K")
    al = np.array([complex(alpha_).real, complex(alpha_).imag])
    be = np.array([complex(beta).real, complex(beta).imag])
    ri, cj = _idx(rows, m), _idx(cols, n)
    rc = lib().oz_ref_zgemm_sub(OP[transA], OP[transB], m, n, k, _p(al), _p(A), lda, _p(B),
                                ldb, _p(be), _p(Cout), ldc, int(s), _p(ri), len(ri), _p(cj),
                                len(cj))
    if rc:
        raise ValueError(f"oz_ref_zgemm_sub failed rc={rc}")
    return Cout


def zgemm_simple(A, B, s, alpha_=1.0, beta=0.0, C=None, transA="N", transB="N", rows=None,
                 cols=None):
    A = np.asfortranarray(A, dtype=np.complex128)
    B = np.asfortranarray(B, dtype=np.complex128)
    m = A.shape[0] if OP[transA] == 0 else A.shape[1]
    k = A.shape[1] if OP[transA] == 0 else A.shape[0]
    n = B.shape[1] if OP[transB] == 0 else B.shape[0]
    if C is None:
        C = np.zeros((m, n), dtype=np.complex128, order="F")
    C = np.asfortranarray(C, dtype=np.complex128)
    return zgemm(transA, transB, m, n, k, alpha_, A, A.shape[0], B, B.shape[0], beta, C, m, s,
                 rows, cols)


def dd_zgemm(transA, transB, m, n, k, A, lda, B, ldb, rows=None, cols=None):
    """Returns (re_hi, re_lo, im_hi, im_lo) as [nr][nc] arrays."""
    A = _c128(A)
    B = _c128(B)
    ri, cj = _idx(rows, m), _idx(cols, n)
    out = [np.zeros((len(ri), len(cj))) for _ in range(4)]
    lib().dd_zgemm_sub(OP[transA], OP[transB], m, n, k, _p(A), lda, _p(B), ldb, _p(ri), len(ri),
                       _p(cj), len(cj), *[_p(o) for o in out])
    return tuple(out)


def zerr_stats(C, rh, rl, ih, il):
    """Complex relative error |C - C_DD| / |C_DD| (modulus), as err_stats."""
    C = np.asarray(C, dtype=np.complex128)
    dr = (C.real - rh) - rl
    di = (C.imag - ih) - il
    diff = np.hypot(dr, di)
    ref = np.hypot(rh, ih)
    nz = ref != 0
    rel = diff[nz] / ref[nz]
    return {"mean_rel": float(rel.mean()) if rel.size else 0.0,
            "max_rel": float(rel.max()) if rel.size else 0.0,
            "nw_max": float(diff.max() / ref.max()) if ref.max() > 0 else float(diff.max()),
            "zero_ref": int((~nz).sum())}


# --- DD reference ------------------------------------------------------------------

def two_sum(a, b):
    hi, lo = ct.c_double(), ct.c_double()
    lib().dd_two_sum(float(a), float(b), ct.byref(hi), ct.byref(lo))
    return hi.value, lo.value


def two_prod(a, b):
    hi, lo = ct.c_double(), ct.c_double()
    lib().dd_two_prod(float(a), float(b), ct.byref(hi), ct.byref(lo))
    return hi.value, lo.value


def dd_gemm(transA, transB, m, n, k, A, lda, B, ldb, rows=None, cols=None):
    """Returns (hi, lo) as [nr][nc] arrays."""
    A = _f64(A)
    B = _f64(B)
    ri, cj = _idx(rows, m), _idx(cols, n)
    hi = np.zeros((len(ri), len(cj)))
    lo = np.zeros((len(ri), len(cj)))
    lib().dd_gemm_sub(OP[transA], OP[transB], m, n, k, _p(A), lda, _p(B), ldb, _p(ri), len(ri),
                      _p(cj), len(cj), _p(hi), _p(lo))
    return hi, lo


def fp64_gemm(transA, transB, m, n, k, A, lda, B, ldb, rows=None, cols=None):
    A = _f64(A)
    B = _f64(B)
    ri, cj = _idx(rows, m), _idx(cols, n)
    out = np.zeros((len(ri), len(cj)))
    lib().fp64_gemm_sub(OP[transA], OP[transB], m, n, k, _p(A), lda, _p(B), ldb, _p(ri),
                        len(ri), _p(cj), len(cj), _p(out))
    return out


def err_stats(C, hi, lo):
    """Relative error of C vs the DD reference: per element
    |C - C_DD| / |C_DD| with C_DD = hi + lo; entries with C_DD == 0 excluded
    (counted).  Returns dict(mean_rel, max_rel, nw_max, zero_ref).
    nw_max = max|C - C_DD| / max|C_DD| (normwise reading)."""
    C = np.asarray(C, dtype=np.float64)
    diff = np.abs((C - hi) - lo)
    ref = np.abs(hi)
    nz = ref != 0
    rel = diff[nz] / ref[nz]
    return {
        "mean_rel": float(rel.mean()) if rel.size else 0.0,
        "max_rel": float(rel.max()) if rel.size else 0.0,
        "nw_max": float(diff.max() / ref.max()) if ref.max() > 0 else float(diff.max()),
        "zero_ref": int((~nz).sum()),
    }
