"""The optional CTA-pair variant of the fused GEMM (OZIMMU_CLUSTER=2: clusters of two CTAs,
A tiles TMA-multicast to both, dummy tile when the column-tile count is odd) must give the
same bits as the default kernel: re-run the DGEMM / ZGEMM / batched parity suites with it
enabled (the variable is read once per process, hence the subprocess)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parity_suites_with_cta_pairs():
    env = dict(os.environ, OZIMMU_CLUSTER="2")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        os.path.join(ROOT, "tests", "test_gpu_zgemm.py"),
                        os.path.join(ROOT, "tests", "test_gpu_batched.py")],
                       env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
