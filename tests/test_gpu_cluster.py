"""The fused GEMM runs by default as CTA pairs (clusters of two CTAs, A tiles TMA-multicast
to both, dummy tile when the column-tile count is odd); OZIMMU_CLUSTER=1 forces single CTAs.
OZIMMU_CLUSTER=4 takes 2 x 2 clusters (B tiles multicast between the two row blocks too).
All must give the same bits: the default suites cover the pairs, this re-runs the DGEMM /
ZGEMM / batched parity suites with single CTAs and with 2 x 2 clusters (the variable is read
once per process, hence the subprocess)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("cl", ["1", "4"])
def test_parity_suites_with_other_cluster_shapes(cl):
    env = dict(os.environ, OZIMMU_CLUSTER=cl)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        os.path.join(ROOT, "tests", "test_gpu_zgemm.py"),
                        os.path.join(ROOT, "tests", "test_gpu_batched.py")],
                       env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
