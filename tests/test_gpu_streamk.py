"""GPU parity of the stream-K schedule of k_oz_gemm (small problems: clusters share the K
loops of the tail units; a split unit's exact int32 partial level sums are added by the last
cluster to finish it, so L_g -- and therefore C -- are the same integers as one CTA over the
whole K, P:353-356 / reading A15).  Children run with the schedule forced on and off
(OZIMMU_SK); every result must be bitwise equal between them and to the CPU oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from streamk_child import CASES  # noqa: E402


def _run(tmp_path, sk):
    out = str(tmp_path / f"sk{sk}.npz")
    env = dict(os.environ)
    env["OZIMMU_SK"] = str(sk)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "streamk_child.py"), out, ROOT],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


def test_streamk_forced_equals_data_parallel_and_oracle(tmp_path):
    on, off = _run(tmp_path, 1), _run(tmp_path, 0)
    for key in on.files:
        assert np.array_equal(on[key], off[key]), key
    for i, (ta, tb, m, n, k, s, phi) in enumerate(CASES):
        A = synth.gen_phi(*((m, k) if ta == "N" else (k, m)), phi, 900 + i)
        B = synth.gen_phi(*((k, n) if tb == "N" else (n, k)), phi, 950 + i)
        Cin = synth.gen_phi(m, n, 0.5, 990 + i)
        rows = None if m * n <= 400_000 else np.r_[0:3, 127:131, m - 3:m]
        ref = O.dgemm(ta, tb, m, n, k, 1.5, A, A.shape[0], B, B.shape[0], -0.5, Cin, m, s,
                      rows=rows)
        got = on[f"C{i}"]
        if rows is None:
            assert np.array_equal(got, ref), i
        else:
            assert np.array_equal(got[rows], ref[rows]), i
        if f"L{i}" in on.files:
            L = O.level_sums(ta, tb, m, n, k, A, A.shape[0], B, B.shape[0], s,
                             rows=None if rows is None else rows)
            gotL = on[f"L{i}"] if rows is None else on[f"L{i}"][:, rows, :]
            assert np.array_equal(gotL, L), i
    Az = synth.gen_phi_complex(300, 200, 0.5, 7)
    Bz = synth.gen_phi_complex(200, 170, 0.5, 8)
    refz = O.zgemm("N", "N", 300, 170, 200, 1.0, Az, 300, Bz, 200, 0.0,
                   np.zeros((300, 170), np.complex128, order="F"), 300, 9)
    assert np.array_equal(on["Z"], refz)
