"""B200-native Ozaki-scheme DGEMM on INT8 tensor cores (arXiv 2306.11975).

The product is the C-ABI library ``libozimmu.so`` (include/ozimmu.h) built from
``csrc/`` for sm_100a; this package is its thin Python binding plus the
multi-GPU driver.  No CPU fallback exists.
"""
from .ozimmu import (BCAST_FN, EXPORTS, Handle, NcclComm, OzimmuError,  # noqa: F401
                     b_slices_bytes, lib, nccl_unique_id, version, workspace_bytes)

__all__ = ["Handle", "NcclComm", "OzimmuError", "lib", "version", "workspace_bytes",
           "b_slices_bytes", "nccl_unique_id", "BCAST_FN", "EXPORTS"]
