"""Seeded random-configuration parity (GPU vs the CPU oracle, bit-exact): shapes that straddle
tile edges (128-row blocks, N_c-column tiles, 128-byte k-blocks, 16-element k padding), every
op combination, slice counts 1..20, phi from 0 to 4, leading-dimension padding and alpha /
beta including 0 -- for DGEMM, ZGEMM and the strided-batched DGEMM with a shared operand.
Each case is drawn from a fixed seed, so a failure names a reproducible configuration."""
import numpy as np
import pytest

import oracle as O
import synth
from gpu_util import dev, host

pytestmark = pytest.mark.gpu

OPS = ["N", "T", "C"]


@pytest.fixture(scope="module")
def h():
    import paper_2306_11975_b200 as oz
    return oz.Handle(0)


def _stored(trans, rows, cols):
    return (rows, cols) if trans == "N" else (cols, rows)


def _dim(rng, edges):
    e = int(rng.choice(edges))
    return max(1, e + int(rng.integers(-2, 3)))


def _case(seed):
    rng = np.random.default_rng(seed)
    m = _dim(rng, [1, 7, 64, 128, 129, 255, 300])
    n = _dim(rng, [1, 16, 32, 48, 64, 97, 200])
    k = _dim(rng, [1, 15, 16, 17, 128, 129, 500, 1100])
    s = int(rng.integers(1, 21))
    ta, tb = str(rng.choice(OPS)), str(rng.choice(OPS))
    phi = float(rng.choice([0.0, 0.1, 0.5, 1.0, 2.0, 4.0]))
    alpha = float(rng.choice([1.0, -0.75, 0.0, 3.5]))
    beta = float(rng.choice([0.0, 1.0, -2.0]))
    pad = [int(rng.integers(0, 4)) for _ in range(3)]
    return m, n, k, s, ta, tb, phi, alpha, beta, pad


@pytest.mark.parametrize("seed", range(24))
def test_dgemm_random_config(h, seed):
    import torch
    m, n, k, s, ta, tb, phi, alpha, beta, pad = _case(1000 + seed)
    ra, ca = _stored(ta, m, k)
    rb, cb = _stored(tb, k, n)
    A = synth.gen_phi(ra + pad[0], ca, phi, 2000 + seed)
    B = synth.gen_phi(rb + pad[1], cb, phi, 3000 + seed)
    C = synth.gen_phi(m + pad[2], n, phi, 4000 + seed)
    lda, ldb, ldc = A.shape[0], B.shape[0], C.shape[0]
    dC = dev(C)
    h.dgemm(ta, tb, m, n, k, alpha, dev(A), lda, dev(B), ldb, beta, dC, ldc, s)
    torch.cuda.synchronize()
    got = host(dC, ldc, n)
    ref = O.dgemm(ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, s)
    assert np.array_equal(got, ref), (m, n, k, s, ta, tb, phi, alpha, beta, pad)


@pytest.mark.parametrize("seed", range(12))
def test_zgemm_random_config(h, seed):
    import torch
    m, n, k, s, ta, tb, phi, alpha, beta, pad = _case(5000 + seed)
    m, n, k = min(m, 150), min(n, 100), min(k, 600)
    rng = np.random.default_rng(6000 + seed)
    za = complex(alpha, float(rng.choice([0.0, 0.5])))
    zb = complex(beta, float(rng.choice([0.0, -1.5])))
    ra, ca = _stored(ta, m, k)
    rb, cb = _stored(tb, k, n)
    A = synth.gen_phi_complex(ra + pad[0], ca, phi, 7000 + seed)
    B = synth.gen_phi_complex(rb + pad[1], cb, phi, 8000 + seed)
    C = synth.gen_phi_complex(m + pad[2], n, phi, 9000 + seed)
    lda, ldb, ldc = A.shape[0], B.shape[0], C.shape[0]

    def zdev(a):
        return torch.from_numpy(np.ascontiguousarray(a.ravel(order="F"))).cuda()
    dC = zdev(C)
    h.zgemm(ta, tb, m, n, k, za, zdev(A), lda, zdev(B), ldb, zb, dC, ldc, s)
    torch.cuda.synchronize()
    got = np.asfortranarray(dC.cpu().numpy().reshape((n, ldc)).T)
    ref = O.zgemm(ta, tb, m, n, k, za, A.ravel(order="F"), lda, B.ravel(order="F"), ldb, zb,
                  C.ravel(order="F"), ldc, s)
    ref = np.asfortranarray(ref.reshape((n, ldc)).T)
    assert np.array_equal(got, ref), (m, n, k, s, ta, tb, phi, za, zb, pad)


@pytest.mark.parametrize("seed", range(6))
def test_dgemm_strided_batched_shared_operand_random(h, seed):
    """A shared (strideA = 0) or B shared (strideB = 0): each item equals its own oracle call."""
    import torch
    rng = np.random.default_rng(11000 + seed)
    m, n, k = int(rng.integers(1, 40)), int(rng.integers(1, 60)), int(rng.integers(1, 300))
    batch, s = int(rng.integers(1, 9)), int(rng.integers(3, 14))
    shared_a = bool(seed % 2)
    A = [synth.gen_phi(m, k, 0.5, 12000 + 10 * seed + (0 if shared_a else b)) for b in range(batch)]
    B = [synth.gen_phi(k, n, 0.5, 13000 + 10 * seed + (b if shared_a else 0)) for b in range(batch)]
    C = [synth.gen_phi(m, n, 0.5, 14000 + 10 * seed + b) for b in range(batch)]
    dA = dev(A[0]) if shared_a else torch.cat([dev(a) for a in A])
    dB = torch.cat([dev(b) for b in B]) if shared_a else dev(B[0])
    dC = torch.cat([dev(c) for c in C])
    h.dgemm_strided_batched("N", "N", m, n, k, 1.25, dA, m, 0 if shared_a else m * k, dB, k,
                            k * n if shared_a else 0, -0.5, dC, m, m * n, batch, s)
    torch.cuda.synchronize()
    for b in range(batch):
        got = host(dC[b * m * n:(b + 1) * m * n], m, n)
        ref = O.dgemm("N", "N", m, n, k, 1.25, A[b], m, B[b], k, -0.5, C[b], m, s)
        assert np.array_equal(got, ref), (b, m, n, k, s, shared_a)
