"""Child process for tests/test_gpu_shim.py: an unmodified PyTorch program doing float64 /
complex128 matmuls on the GPU.  Run under LD_PRELOAD=libozimmu_cublas_shim.so its cuBLAS
GEMMs execute on the INT8 Ozaki path.  Inputs come from synth (seeded); the
outputs are saved to the .npz named by argv[1]."""
import sys

import numpy as np
import torch

sys.path.insert(0, sys.argv[2])
import synth  # noqa: E402


def main(out):
    m, n, k = 96, 80, 200
    A = synth.gen_phi(m, k, 1.0, 1)
    B = synth.gen_phi(k, n, 1.0, 2)
    C = (torch.from_numpy(np.ascontiguousarray(A)).cuda() @
         torch.from_numpy(np.ascontiguousarray(B)).cuda())
    Az = synth.gen_phi_complex(m, k, 0.5, 3)
    Bz = synth.gen_phi_complex(k, n, 0.5, 4)
    Cz = (torch.from_numpy(np.ascontiguousarray(Az)).cuda() @
          torch.from_numpy(np.ascontiguousarray(Bz)).cuda())
    batch, bm, bn, bk = 3, 32, 24, 48
    Ab = np.ascontiguousarray(np.stack([synth.gen_phi(bm, bk, 1.0, 10 + b) for b in range(batch)]))
    Bb = np.ascontiguousarray(np.stack([synth.gen_phi(bk, bn, 1.0, 20 + b) for b in range(batch)]))
    Cb = torch.bmm(torch.from_numpy(Ab).cuda(), torch.from_numpy(Bb).cuda())
    torch.cuda.synchronize()
    # the shim's own counters (present only when it is preloaded)
    counters = np.array([-1, -1], dtype=np.int64)
    try:
        import ctypes as ct
        fn = ct.CDLL(None).ozimmu_shim_counters
        a, b = ct.c_longlong(), ct.c_longlong()
        fn(ct.byref(a), ct.byref(b))
        counters = np.array([a.value, b.value], dtype=np.int64)
    except (AttributeError, OSError):
        pass
    np.savez(out, C=C.cpu().numpy(), Cz=Cz.cpu().numpy(), Cb=Cb.cpu().numpy(),
             counters=counters)


if __name__ == "__main__":
    main(sys.argv[1])
