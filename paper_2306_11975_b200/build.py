"""Build libozimmu.so (the C-ABI library) in-tree for sm_100a with nvcc.

The .so lands next to this file so it travels with gpurun snapshots; the
static CUDA runtime is linked in, the driver API is reached through
cudaGetDriverEntryPoint, so the library loads on machines without a GPU
(calls then fail with OZIMMU_ERR_CUDA).
"""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libozimmu.so")
SOURCES = ["api.cu", "split.cu", "igemm.cu"]
HEADERS = ["internal.h", "ptx.cuh", os.path.join("..", "..", "include", "ozimmu.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-DOZIMMU_BUILD"]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    srcs = [os.path.join(CSRC, f) for f in SOURCES]
    cmd = [NVCC] + FLAGS + (["-Xptxas", "-v"] if verbose else []) + \
        ["-shared", "-o", LIB] + srcs
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force=True, verbose="-v" in sys.argv))
