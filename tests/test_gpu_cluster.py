"""The fused GEMM runs by default as CTA pairs (clusters of two CTAs, A tiles TMA-multicast
to both, dummy tile when the column-tile count is odd); OZIMMU_CLUSTER=1 forces single CTAs.
Both must give the same bits: the default suites cover the pairs, this re-runs the DGEMM /
ZGEMM / batched parity suites with single CTAs (the variable is read once per process,
hence the subprocess)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parity_suites_with_single_ctas():
    env = dict(os.environ, OZIMMU_CLUSTER="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        os.path.join(ROOT, "tests", "test_gpu_zgemm.py"),
                        os.path.join(ROOT, "tests", "test_gpu_batched.py")],
                       env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
