"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no splitting, no products, no
accumulation) -- only the input distributions of the paper's experiments, so
that both sides see identical bytes.

gen_phi: the paper's exponent-range workload (s4.2.1):
    A_ij, B_ij = uniform(-0.5, 0.5) * exp(phi * normal(0, 1))
The paper gives no RNG (SPEC notes it); we use numpy's PCG64 via
``default_rng(seed)``: first ``rows*cols`` uniforms in [0,1), then
``rows*cols`` standard normals, both in column-major element order
(element (i, j) is draw number i + j*rows).  Output is a Fortran-ordered
float64 array (BLAS column-major).
"""
import numpy as np

# Seeds of the BASELINE.json configs.
CONFIG_SEEDS = {
    "C1": (101, 102, 103),
    "C2": (201, 211),        # + phi index
    "C3": (301, 302),
    "C4": (401, 402),
}


def gen_phi(rows: int, cols: int, phi: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    n = rows * cols
    u = rng.random(n)
    z = rng.standard_normal(n)
    x = (u - 0.5) * np.exp(phi * z)
    return np.asfortranarray(x.reshape((cols, rows)).T)


def gen_uniform(rows: int, cols: int, lo: float, hi: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    x = lo + (hi - lo) * rng.random(rows * cols)
    return np.asfortranarray(x.reshape((cols, rows)).T)


def gen_normal(rows: int, cols: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(rows * cols)
    return np.asfortranarray(x.reshape((cols, rows)).T)


def gen_int(rows: int, cols: int, lo: int, hi: int, seed: int) -> np.ndarray:
    """Small integers stored as float64 (exact-result workloads)."""
    rng = np.random.default_rng(seed)
    x = rng.integers(lo, hi + 1, rows * cols).astype(np.float64)
    return np.asfortranarray(x.reshape((cols, rows)).T)


def gen_dyadic(rows: int, cols: int, bits: int, emin: int, emax: int, seed: int) -> np.ndarray:
    """Random dyadic rationals  +-(odd <= 2^bits) * 2^e,  e in [emin, emax]."""
    rng = np.random.default_rng(seed)
    n = rows * cols
    mant = rng.integers(1, 2 ** bits, n)
    e = rng.integers(emin, emax + 1, n)
    sgn = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    x = sgn * np.ldexp(mant.astype(np.float64), e)
    return np.asfortranarray(x.reshape((cols, rows)).T)
