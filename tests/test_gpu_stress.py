"""Determinism under shifted timing: the fused GEMM's two MMA issuers, CTA-pair multicast and
mbarrier rings must give identical bits on every repetition, also with the smallest A ring
(OZIMMU_A_STAGES=2, which maximises slot reuse and exposed a phase-aliasing race of odd
rings) and with single CTAs / 2x2 clusters (read once per process, hence subprocesses)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"OZIMMU_A_STAGES": "2"}, {"OZIMMU_CLUSTER": "1"},
                                 {"OZIMMU_CLUSTER": "4", "OZIMMU_A_STAGES": "2"}])
def test_repeated_calls_identical_bits(env):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stress.py"), "3"],
                       env=dict(os.environ, **env), capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "STRESS OK" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]
