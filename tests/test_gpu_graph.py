"""A fixed-s ozimmu_dgemm call can be captured into a CUDA graph (torch.cuda.CUDAGraph on the
handle's stream) and replayed: every replay gives the same bits as the eager call, and the
replay picks up new input values written in place (the graph holds pointers, not data)."""
import numpy as np
import pytest

import synth
from gpu_util import dev, host

pytestmark = pytest.mark.gpu


def test_dgemm_cuda_graph_replay_bitwise():
    import torch
    import paper_2306_11975_b200 as oz
    m, n, k, s = 700, 520, 900, 9
    A1, B1 = synth.gen_phi(m, k, 0.5, 61), synth.gen_phi(k, n, 0.5, 62)
    A2, B2 = synth.gen_phi(m, k, 1.0, 63), synth.gen_phi(k, n, 1.0, 64)
    h = oz.Handle(0)
    dA, dB = dev(A1), dev(B1)
    dC = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    side = torch.cuda.Stream()
    h.set_stream(side)
    with torch.cuda.stream(side):
        h.dgemm("N", "N", m, n, k, 1.0, dA, m, dB, k, 0.0, dC, m, s)  # warm-up: workspace
    torch.cuda.synchronize()
    eager1 = host(dC, m, n).copy()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        h.dgemm("N", "N", m, n, k, 1.0, dA, m, dB, k, 0.0, dC, m, s)
    dC.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(host(dC, m, n), eager1)
    # new inputs in the same buffers: the replay computes the new product
    dA.copy_(dev(A2))
    dB.copy_(dev(B2))
    g.replay()
    torch.cuda.synchronize()
    got2 = host(dC, m, n).copy()
    with torch.cuda.stream(side):
        h.dgemm("N", "N", m, n, k, 1.0, dA, m, dB, k, 0.0, dC, m, s)
    torch.cuda.synchronize()
    assert np.array_equal(got2, host(dC, m, n))
    h.close()
