"""Helpers for the -m gpu parity tests: move column-major numpy matrices to the
device as flat buffers and back.  (No method arithmetic here.)"""
import numpy as np


def dev(a, dtype=None):
    """Column-major (Fortran-order) flattening of a numpy array -> 1-D CUDA tensor."""
    import torch
    flat = np.asarray(a).ravel(order="F")
    if dtype is not None:
        flat = flat.astype(dtype)
    return torch.from_numpy(np.ascontiguousarray(flat)).cuda()


def host(t, rows, cols):
    """1-D device buffer holding a column-major rows x cols matrix -> Fortran numpy array."""
    x = t.detach().cpu().numpy()
    return np.asfortranarray(x[: rows * cols].reshape((cols, rows)).T)


def empty(n, dtype):
    import torch
    return torch.empty(n, dtype=dtype, device="cuda")


def ulp_dist(a, b):
    """Elementwise distance in units in the last place (0 for equal, +-0 equal, NaN==NaN)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    ia = a.view(np.int64).copy()
    ib = b.view(np.int64).copy()
    # map to a monotone integer line
    ia = np.where(ia < 0, np.int64(-0x8000000000000000) - ia, ia)
    ib = np.where(ib < 0, np.int64(-0x8000000000000000) - ib, ib)
    with np.errstate(over="ignore"):
        d = np.abs((ia - ib).astype(np.float64))
    both_nan = np.isnan(a) & np.isnan(b)
    d = np.where(both_nan, 0.0, d)
    d = np.where(np.isnan(a) ^ np.isnan(b), np.inf, d)
    return d
