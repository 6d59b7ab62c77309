"""GPU parity of the one-read slicing kernel (k_split_fused: exponent scan and digits of a
panel in one persistent launch, slice tiles waiting on their panel's scan tiles; SplitInt,
Alg. 4, readings A3-A5/A11).  Children run with the fused kernel at its default
panel size, with tiny panels (many panels, ragged last panel, scans and slices of different
panels interleaved) and with the per-operand kernels (OZIMMU_SPLIT_FUSED=0,
OZIMMU_SPLIT_SMALL_MB=0, the base); the DGEMMs also run with both operands sliced in one
clustered launch (k_split_small, the default for small calls, here also up to 512 MB); the
GEMM cases also
run with one TMEM accumulator instead of two (OZIMMU_ACC2=0).  Planes, exponents and C must
be bitwise equal across the variants and to the CPU oracle."""
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
from split_child import DGEMMS, SPLITS, ZGEMMS, split_matrix  # noqa: E402

VARIANTS = {"two_launch": {"OZIMMU_SPLIT_FUSED": "0", "OZIMMU_SPLIT_SMALL_MB": "0"},
            "default": {},
            "fused": {"OZIMMU_SPLIT_FUSED": "1"},
            "fused_small_panels": {"OZIMMU_SPLIT_FUSED": "1", "OZIMMU_SPLIT_PANEL_KB": "24"},
            "fused_bps2": {"OZIMMU_SPLIT_FUSED": "1", "OZIMMU_SPLIT_FUSED_BPS": "2"},
            # both operands of a DGEMM in one launch (k_split_small) up to 512 MB of input and
            # k_pad <= 2048 (clusters of up to 16 CTAs)
            "small_one_launch": {"OZIMMU_SPLIT_SMALL_MB": "512", "OZIMMU_SPLIT_SMALL_K": "2048"},
            # small strided operands: scan + slice kernels instead of the clustered one-launch
            # kernel (k_split_strided_cl, the default for k_pad <= 2048)
            "no_cluster_split": {"OZIMMU_SPLIT_CL_MB": "0"},
            # GEMM side: one TMEM accumulator buffer instead of two for short K (s <= 8)
            "one_acc": {"OZIMMU_ACC2": "0"}}


@pytest.fixture(scope="module")
def runs(tmp_path_factory):
    out = {}
    d = tmp_path_factory.mktemp("split")
    for name, extra in VARIANTS.items():
        env = dict(os.environ)
        env.update(extra)
        path = str(d / f"{name}.npz")
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "split_child.py"), path,
                            ROOT], env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        out[name] = np.load(path)
    return out


def test_variants_bitwise_equal(runs):
    base = runs["two_launch"]
    for name in VARIANTS:
        for key in base.files:
            assert np.array_equal(runs[name][key], base[key]), (name, key)


def test_split_vs_oracle(runs):
    got = runs["fused_small_panels"]
    for i, (op, is_rows, rows, kdim, s) in enumerate(SPLITS):
        if is_rows:
            shape = (rows, kdim) if op == "N" else (kdim, rows)
            d_ref, E_ref, bad = O.split_opA(split_matrix(shape, 500 + i), op, rows, kdim,
                                            shape[0], s)
        else:
            shape = (kdim, rows) if op == "N" else (rows, kdim)
            d_ref, E_ref, bad = O.split_opB(split_matrix(shape, 500 + i), op, kdim, rows,
                                            shape[0], s)
        assert not bad.any()
        assert np.array_equal(got[f"E{i}"], E_ref), i
        assert np.array_equal(got[f"P{i}"], d_ref), i


def test_gemms_vs_oracle(runs):
    got = runs["fused_small_panels"]
    for i, (ta, tb, m, n, k, s) in enumerate(DGEMMS):
        A = synth.gen_phi(*((m, k) if ta == "N" else (k, m)), 1.0, 600 + i)
        B = synth.gen_phi(*((k, n) if tb == "N" else (n, k)), 1.0, 650 + i)
        Cin = synth.gen_phi(m, n, 0.5, 690 + i)
        ref = O.dgemm(ta, tb, m, n, k, 1.5, A, A.shape[0], B, B.shape[0], -0.5, Cin, m, s)
        assert np.array_equal(got[f"D{i}"], ref), i
    for i, (ta, tb, m, n, k, s) in enumerate(ZGEMMS):
        A = synth.gen_phi_complex(*((m, k) if ta == "N" else (k, m)), 0.5, 700 + i)
        B = synth.gen_phi_complex(*((k, n) if tb == "N" else (n, k)), 0.5, 750 + i)
        Cin = synth.gen_phi_complex(m, n, 0.5, 790 + i)
        ref = O.zgemm(ta, tb, m, n, k, 0.75 - 1.25j, A, A.shape[0], B, B.shape[0], 2.0j, Cin, m, s)
        assert np.array_equal(got[f"Z{i}"], ref), i
