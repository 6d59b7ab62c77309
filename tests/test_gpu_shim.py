"""GPU test of the LD_PRELOAD cuBLAS shim (NEXT row f3): "Intercepting cuBLAS
double-precision GEMM function calls and executing INT8-AUTO instead. We use an
environmental variable LD_PRELOAD to realize it.".

An unmodified PyTorch program (tests/shim_child.py: float64 mm, complex128 mm, float64 bmm)
runs with the shim preloaded; the shim's log proves each call was intercepted, and every
intercepted result is bit-exact against the oracle evaluated on the call the log records
(fixed s, and INT8-AUTO with the oracle's own AUTO choice)."""
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "paper_2306_11975_b200", "libozimmu_cublas_shim.so")
LOG = re.compile(r"\[ozimmu shim\] (\w+) ta=(\w) tb=(\w) m=(\d+) n=(\d+) k=(\d+) batch=(\d+) "
                 r"-> (.+) \(s=(\d+)\)")


def _run(tmp_path, env_extra):
    out = str(tmp_path / "out.npz")
    env = dict(os.environ)
    env.update(env_extra)
    env["LD_PRELOAD"] = SHIM
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "shim_child.py"), out, ROOT],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    calls = [m.groups() for m in map(LOG.search, r.stderr.splitlines()) if m]
    return np.load(out), calls


def _col(X):
    """The column-major operand cuBLAS sees for a row-major torch matrix X: X^T."""
    return np.asfortranarray(np.asarray(X).T)


def _s_auto(ta, tb, m, n, k, A, lda, B, ldb, mode):
    """The oracle's INT8-AUTO choice under the shim's rule (mode 'acc' = reading A18, the
    default; 'loss' = the paper's T = 0 rule, reading A17)."""
    if mode == "loss":
        return O.auto_splits(ta, tb, m, n, k, A, lda, B, ldb, 0.0, 18)
    return O.auto_splits_acc(ta, tb, m, n, k, A, lda, B, ldb, 1.0, 18)[0]


def _check_calls(res, calls, fixed_s, mode="acc"):
    assert [c[0] for c in calls] == ["cublasDgemm_v2", "cublasZgemm_v2",
                                     "cublasDgemmStridedBatched"], calls
    # row-major C = A B reaches cuBLAS as C^T = B^T A^T: ta = tb = N, (m, n) swapped
    m, n, k = 96, 80, 200
    for fn, ta, tb, cm, cn, ck, batch, status, s in calls:
        assert (ta, tb) == ("N", "N") and "success" in status.lower(), (fn, status)
    fn, _, _, cm, cn, ck, _, _, s = calls[0]
    assert (int(cm), int(cn), int(ck)) == (n, m, k)
    A, B = synth.gen_phi(m, k, 1.0, 1), synth.gen_phi(k, n, 1.0, 2)
    s = int(s)
    if fixed_s:
        assert s == fixed_s
    else:
        assert s == _s_auto("N", "N", n, m, k, _col(B), n, _col(A), k, mode)
    ref = O.dgemm("N", "N", n, m, k, 1.0, _col(B), n, _col(A), k, 0.0,
                  np.zeros((n, m), order="F"), n, s)
    assert np.array_equal(res["C"], ref.T)

    s = int(calls[1][8])
    Az, Bz = synth.gen_phi_complex(m, k, 0.5, 3), synth.gen_phi_complex(k, n, 0.5, 4)
    if fixed_s:
        assert s == fixed_s
    ref = O.zgemm("N", "N", n, m, k, 1.0, _col(Bz), n, _col(Az), k, 0.0,
                  np.zeros((n, m), np.complex128, order="F"), n, s)
    assert np.array_equal(res["Cz"], ref.T)

    batch, bm, bn, bk = 3, 32, 24, 48
    _, _, _, cm, cn, ck, cb, _, _ = calls[2]
    assert (int(cm), int(cn), int(ck), int(cb)) == (bn, bm, bk, batch)
    for b in range(batch):
        Ab, Bb = synth.gen_phi(bm, bk, 1.0, 10 + b), synth.gen_phi(bk, bn, 1.0, 20 + b)
        sb = fixed_s or _s_auto("N", "N", bn, bm, bk, _col(Bb), bn, _col(Ab), bk, mode)
        ref = O.dgemm("N", "N", bn, bm, bk, 1.0, _col(Bb), bn, _col(Ab), bk, 0.0,
                      np.zeros((bn, bm), order="F"), bn, sb)
        assert np.array_equal(res["Cb"][b], ref.T), b
    # every intercepted call ran on libozimmu: nothing fell through to cuBLAS
    assert list(res["counters"]) == [3, 0], res["counters"]


def test_shim_fixed_slices(tmp_path):
    res, calls = _run(tmp_path, {"OZIMMU_SHIM_LOG": "1", "OZIMMU_SHIM_SLICES": "9"})
    _check_calls(res, calls, 9)


def test_shim_int8_auto(tmp_path):
    """Default: INT8-AUTO with the accuracy-targeted rule (reading A18, tau = 1)."""
    env = {"OZIMMU_SHIM_LOG": "1"}
    res, calls = _run(tmp_path, env)
    _check_calls(res, calls, None, "acc")


def test_shim_int8_auto_loss_rule(tmp_path):
    """OZIMMU_SHIM_AUTO=loss: the paper's rule with T = 0 (the lossless setting)."""
    res, calls = _run(tmp_path, {"OZIMMU_SHIM_LOG": "1", "OZIMMU_SHIM_AUTO": "loss"})
    _check_calls(res, calls, None, "loss")


def test_shim_counts_fall_through(tmp_path):
    """A call libozimmu rejects (s > OZIMMU_MAX_SLICES) goes to cuBLAS, is counted and is
    reported on stderr -- never silent."""
    out = str(tmp_path / "out.npz")
    env = dict(os.environ)
    env.update({"OZIMMU_SHIM_SLICES": "99", "LD_PRELOAD": SHIM})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "shim_child.py"), out, ROOT],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = np.load(out)
    assert list(res["counters"]) == [0, 3], res["counters"]
    assert "WARNING cublasDgemm_v2 ran on cuBLAS FP64 instead" in r.stderr


def test_shim_disabled_forwards_to_cublas(tmp_path):
    res, calls = _run(tmp_path, {"OZIMMU_SHIM_LOG": "1", "OZIMMU_SHIM_DISABLE": "1"})
    assert calls == []
    assert list(res["counters"]) == [0, 3]
    m, n, k = 96, 80, 200
    A, B = synth.gen_phi(m, k, 1.0, 1), synth.gen_phi(k, n, 1.0, 2)
    ref = A @ B
    assert np.max(np.abs(res["C"] - ref)) <= 1e-13 * np.max(np.abs(A) @ np.abs(B))
