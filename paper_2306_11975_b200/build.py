"""Build libozimmu.so (the C-ABI library) in-tree for sm_100a with nvcc.

The .so lands next to this file so it travels with gpurun snapshots; the
static CUDA runtime is linked in and the driver API is reached through
cudaGetDriverEntryPoint, so the library loads on machines without a GPU
(calls then fail with OZIMMU_ERR_CUDA).  Translation units are compiled to
objects in parallel (the fused GEMM is instantiated for s = 1..32 across
igemm_inst_*.cu), then linked.
"""
import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# development variants: OZIMMU_VARIANT=<name> OZIMMU_EXTRA_FLAGS="-D..." builds
# variants/libozimmu_<name>.so (selected at run time with OZIMMU_LIB=...); default: the product
VARIANT = os.environ.get("OZIMMU_VARIANT", "")
OBJ = os.path.join(HERE, "build" + ("_" + VARIANT if VARIANT else ""))
LIB = (os.path.join(HERE, "variants", f"libozimmu_{VARIANT}.so") if VARIANT
       else os.path.join(HERE, "libozimmu.so"))
SHIM = os.path.join(HERE, "libozimmu_cublas_shim.so")
SHIM_SRC = os.path.join(CSRC, "shim", "cublas_shim.cpp")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-DOZIMMU_BUILD", "-I", INCLUDE] + os.environ.get("OZIMMU_EXTRA_FLAGS", "").split()


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(INCLUDE, "*.h")))


def _obj(src):
    return os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    hdrs = headers() + [os.path.abspath(__file__)]
    jobs = [s for s in sources() if force or _stale(_obj(s), [s] + hdrs)]

    def compile_one(src):
        cmd = [NVCC] + FLAGS + (["-Xptxas", "-v"] if verbose else []) + \
            ["-c", src, "-o", _obj(src)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            print(r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"nvcc failed on {src}")

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(compile_one, jobs))
    objs = [_obj(s) for s in sources()]
    if force or jobs or _stale(LIB, objs):
        subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB]
                       + objs, check=True)
    if VARIANT:
        return LIB
    # f3: LD_PRELOAD cuBLAS shim (host C++ only; resolves libozimmu.so next to itself)
    if force or _stale(SHIM, [SHIM_SRC, LIB] + hdrs):
        subprocess.run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-fvisibility=hidden",
                        "-I", INCLUDE, "-I", "/usr/local/cuda/include", "-o", SHIM, SHIM_SRC,
                        "-L", HERE, "-lozimmu", "-Wl,-rpath,$ORIGIN", "-ldl"], check=True)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force="-f" in sys.argv or "-v" in sys.argv, verbose="-v" in sys.argv))
