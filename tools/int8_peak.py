"""Library INT8 / FP8 tensor-core throughput on this B200 (a roofline denominator).

Measures cuBLASLt INT8 GEMM (torch._int_mm, i8 x i8 -> i32) and FP8 e4m3 GEMM
(torch._scaled_mm) the way MEASURED_PEAKS.json measures bf16: best of 10 CUDA-event-timed
calls (burst) and back to back for ~4 s (sustained), with nvidia-smi clocks/power sampled
during the sustained loop.  Operands are uniform random in [-127, 127] (INT8) -- the value
distribution of the Ozaki digit planes -- and zeros as a power-floor contrast.

    python tools/int8_peak.py [N ...]     (default 8192 16384)
prints one JSON object per line.
"""
import json
import os
import subprocess
import sys
import threading
import time

import torch


def smi():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                              "-i", "0"], capture_output=True, text=True, timeout=5).stdout.strip()
        a, b = out.split(",")
        return float(a), float(b)
    except Exception:
        return None, None


def run(fn, ops, secs=4.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(10):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    # sustained: back to back for `secs`, clocks sampled by a side thread (never stalls the GPU)
    samples = []
    stop = threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append(smi())
            time.sleep(0.2)
    th = threading.Thread(target=sampler, daemon=True)
    n = max(4, int(secs * 1e3 / best))
    th.start()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / n
    clk = sorted(s[0] for s in samples if s[0])
    pw = sorted(s[1] for s in samples if s[1])
    return {"burst_tops": ops / best / 1e9, "sustained_tops": ops / ms / 1e9,
            "sm_mhz_median": clk[len(clk) // 2] if clk else None,
            "power_w_median": pw[len(pw) // 2] if pw else None}


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [8192, 16384]
    torch.manual_seed(0)
    for N in sizes:
        ops = 2.0 * N ** 3
        a = torch.randint(-127, 128, (N, N), dtype=torch.int8, device="cuda")
        b = torch.randint(-127, 128, (N, N), dtype=torch.int8, device="cuda").t()  # col-major B
        r = run(lambda: torch._int_mm(a, b), ops)
        print(json.dumps({"N": N, "op": "cublasLt int8 (torch._int_mm) random [-127,127]", **r}), flush=True)
        z = torch.zeros_like(a)
        zb = torch.zeros_like(a).t()
        r = run(lambda: torch._int_mm(z, zb), ops)
        print(json.dumps({"N": N, "op": "cublasLt int8 (torch._int_mm) zeros", **r}), flush=True)
        try:
            fa = (torch.rand(N, N, device="cuda") * 2 - 1).to(torch.float8_e4m3fn)
            fb = (torch.rand(N, N, device="cuda") * 2 - 1).to(torch.float8_e4m3fn).t()
            one = torch.ones((), device="cuda")
            r = run(lambda: torch._scaled_mm(fa, fb, one, one, out_dtype=torch.bfloat16), ops)
            print(json.dumps({"N": N, "op": "cublasLt fp8 e4m3 (torch._scaled_mm) random", **r}), flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"N": N, "op": "fp8", "error": str(e)[:200]}), flush=True)
        del a, b, z, zb
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
