"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every
symbol include/ozimmu.h declares, and its synchronous argument validation and
size queries behave as documented (no compute calls without a GPU)."""
import ctypes as ct
import os
import re

import pytest

import paper_2306_11975_b200 as oz
from paper_2306_11975_b200 import ozimmu as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "ozimmu.h")).read()
    return sorted(set(re.findall(r"OZIMMU_API\s+[\w\s\*]+?\b(ozimmu_\w+)\s*\(", src)))


def test_header_declares_exports():
    assert _declared() == sorted(B.EXPORTS)


def test_library_loads_and_exports_all_symbols():
    L = oz.lib()
    for name in _declared():
        assert hasattr(L, name), name
    assert oz.version() == 100


def test_status_strings():
    L = oz.lib()
    assert L.ozimmu_status_string(0) == b"OZIMMU_SUCCESS"
    assert L.ozimmu_status_string(2) == b"OZIMMU_ERR_UNSUPPORTED"


def test_workspace_bytes_formula():
    # s (m + n) k_pad INT8 planes + exponents (+ alignment); k = 1000 -> k_pad = 1008
    s, m, n, k = 9, 300, 200, 1000
    wb = oz.workspace_bytes("N", "N", m, n, k, s)
    assert wb >= s * (m + n) * 1008 + 4 * (m + n)
    assert wb < s * (m + n) * 1008 + 4 * (m + n) + 8 * 1024 * 1024
    assert oz.workspace_bytes("N", "N", m, n, k, 0) == 0
    assert oz.workspace_bytes("N", "N", m, n, k, 33) == 0
    assert oz.workspace_bytes("N", "N", -1, n, k, 9) == 0
    # the paper's memory figure at the headline size: 9 x 2 x 16384^2 B = 4.8 GB
    big = oz.workspace_bytes("N", "N", 16384, 16384, 16384, 9)
    assert 9 * 2 * 16384 ** 2 <= big <= 9 * 2 * 16384 ** 2 + 128 * 1024 * 1024


def test_b_slices_bytes():
    assert oz.b_slices_bytes(100, 30, 9) >= 9 * 100 * 32 + 400
    assert oz.b_slices_bytes(100, 30, 0) == 0


def test_create_without_gpu_fails_cleanly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(oz.OzimmuError) as e:
        oz.Handle(0)
    assert e.value.code == 4  # OZIMMU_ERR_CUDA


def test_null_handle_validation():
    L = oz.lib()
    one = ct.byref(ct.c_double(1.0))
    # NULL handle -> NOT_INITIALIZED, before anything else
    assert L.ozimmu_dgemm(None, 0, 0, 4, 4, 4, one, 1, 4, 1, 4, one, 1, 4, 9) == 5
    assert L.ozimmu_set_stream(None, None) == 5
    assert L.ozimmu_destroy(None) == 0


def test_cublas_shim_exports():
    """NEXT row f3: the LD_PRELOAD shim defines exactly the cuBLAS GEMMs it interposes (plus its
    counters) and loads without a GPU (resolving libozimmu.so next to itself)."""
    import ctypes
    import subprocess
    shim = os.path.join(os.path.dirname(B.__file__), "libozimmu_cublas_shim.so")
    assert os.path.exists(shim), "run __graft_entry__.build()"
    out = subprocess.run(["nm", "-D", "--defined-only", shim], capture_output=True, text=True,
                         check=True).stdout
    defined = sorted(l.split()[-1] for l in out.splitlines() if " T " in l)
    assert defined == sorted(["cublasDgemm_v2", "cublasZgemm_v2", "cublasDgemmStridedBatched",
                              "cublasZgemmStridedBatched", "ozimmu_shim_counters"])
    L = ctypes.CDLL(shim)
    a, b = ctypes.c_longlong(7), ctypes.c_longlong(7)
    L.ozimmu_shim_counters(ctypes.byref(a), ctypes.byref(b))
    assert (a.value, b.value) == (0, 0)
