#!/usr/bin/env python3
"""bench.py -- effective DGEMM TFLOP/s (2mnk/t) of the B200-native INT8 Ozaki scheme.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4|C3] [--impl ours|reference]

One step = one whole Ozaki DGEMM (slice B, slice A, fused tcgen05 INT8 GEMMs + FP64
epilogue; for N > 1 also the broadcast of B's INT8 planes) on the BASELINE.json
workload.  Default workload C4: m = n = k = 16384, phi = 0.5, s = 9 (the
FP64-equivalent slice count), C row-block partitioned over N GPUs (strong
scaling).  Prints ONE JSON line on rank 0.  See DESIGN.md s7.
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

WORKLOADS = {
    "C4": dict(m=16384, n=16384, k=16384, phi=0.5, s=9, seeds=(401, 402),
               desc="C4: DGEMM m=n=k=16384, phi=0.5, s=9 (FP64-equivalent), C row blocks over N "
                    "GPUs + NCCL broadcast of B's INT8 slices"),
    "C3": dict(m=8192, n=8192, k=8192, phi=0.5, s=9, seeds=(301, 302),
               desc="C3: DGEMM m=n=k=8192, phi=0.5, s=9 (FP64-equivalent)"),
    # ZGEMM of BASELINE config 5: one d-qubit gate on an N-qubit state vector,
    # matmul-(2^(N-d), 2^d, 2^d), N = 28, d = 12, s = 12 (the T = 0 AUTO choice
    # for the paper's circuits was INT8x12/13)
    "C5": dict(m=2 ** 16, n=2 ** 12, k=2 ** 12, phi=0.1, s=12, seeds=(501, 502), complex=True,
               desc="C5: ZGEMM matmul-(2^16, 2^12, 2^12) = one 12-qubit Haar gate on a 28-qubit "
                    "state vector, s=12"),
    # the same gate on qubits o..o+d-1 of the middle of the register (o = 4): the state is a
    # (2^(N-d-o), 2^d, 2^o) tensor and the gate a strided-batched ZGEMM with a shared U:
    # batch 2^12 of matmul-(2^o, 2^d, 2^d) (column-major view), one fused GEMM here
    "C5B": dict(m=2 ** 4, n=2 ** 12, k=2 ** 12, batch=2 ** 12, phi=0.1, s=12, seeds=(511, 512),
                complex=True,
                desc="C5B: batched ZGEMM, 12-qubit Haar gate on qubits 4..15 of a 28-qubit state: "
                     "batch 4096 x matmul-(16, 4096, 4096) with shared U, s=12"),
}
# SMs kept free of the GEMM for the NCCL broadcast of the next B chunk (N > 1)
RESERVE_SMS = int(os.environ.get("OZIMMU_RESERVE_SMS", "8"))
METRIC = "effective DGEMM TFLOP/s (2mnk/t) vs cuBLAS DGEMM at 1/2/4/8 B200; max rel err"
INT8_PEAK_NOTE = ("INT8 dense peak = 2 x measured bf16 cuBLAS (nominal 4.5/2.25 POPS ratio); "
                  "'sustained' (seconds-long loop under the power cap) used: the kernel is timed "
                  "inside long back-to-back steps")


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def library_int8_context():
    """cuBLASLt INT8 / FP8 throughput measured on this pool's B200s by tools/int8_peak.py
    (16384^3, random operands; committed log), the library rate our INT8 work compares to."""
    p = os.path.join(ROOT, "profiles", "r01b", "cublaslt_int8_fp8_16384.log")
    out = {"source": "profiles/r01b/cublaslt_int8_fp8_16384.log (tools/int8_peak.py)"}
    try:
        for line in open(p):
            d = json.loads(line)
            if "error" in d:
                continue
            key = "cublaslt_int8" if "int8" in d["op"] and "random" in d["op"] else (
                "cublaslt_fp8" if "fp8" in d["op"] else None)
            if key:
                out[key + "_burst_tops"] = round(d["burst_tops"], 1)
                out[key + "_sustained_tops"] = round(d["sustained_tops"], 1)
    except (OSError, ValueError, KeyError):
        return None
    return out


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                c = [x.strip() for x in line.split(",")]
                if len(c) < 9:
                    continue
                try:
                    sm.append(float(c[1]))
                    smax.append(float(c[2]))
                    power.append(float(c[3]))
                except ValueError:
                    continue
                for nm, v in zip(names, c[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": float(np.median(power))}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline_sample(A, B, k, s, target_s=15.0):
    """Time the oracle (as it stands, test infrastructure) on a bounded sample of the
    workload: `rows` rows x `cols` columns of C (rows of A / columns of B gathered whole,
    so exponents are the workload's).  Returns (value TFLOP/s, seconds, sample desc, C)."""
    import oracle as O
    m, n = A.shape[0], B.shape[1]
    rng = np.random.default_rng(7)
    # calibrate on a tiny block, then size the sample for ~target_s of CPU work
    # (16 x 256 outputs: enough work per call for the oracle's threads; an 8 x 32 block
    # overestimated the per-output cost about 4x, so the sample ran ~4 s instead of ~15 s)
    cr, cc = min(m, 16), min(n, 256)
    r0 = rng.choice(m, cr, replace=False)
    c0 = rng.choice(n, cc, replace=False)
    t = time.perf_counter()
    O.dgemm("N", "N", cr, cc, k, 1.0, np.asfortranarray(A[r0]), cr, np.asfortranarray(B[:, c0]),
            k, 0.0, np.zeros((cr, cc), order="F"), cr, s)
    dt = max(time.perf_counter() - t, 1e-3)
    per_elem = dt / (cr * cc)
    nel = max(256, int(target_s / per_elem))
    rows_n = int(min(m, max(8, 2 ** int(np.log2(max(8, np.sqrt(nel / 8)))))))
    cols_n = int(min(n, max(32, nel // rows_n)))
    rows = np.sort(rng.choice(m, rows_n, replace=False))
    cols = np.sort(rng.choice(n, cols_n, replace=False))
    As, Bs = np.asfortranarray(A[rows]), np.asfortranarray(B[:, cols])
    t = time.perf_counter()
    Cs = O.dgemm("N", "N", rows_n, cols_n, k, 1.0, As, rows_n, Bs, k, 0.0,
                 np.zeros((rows_n, cols_n), order="F"), rows_n, s)
    dt = time.perf_counter() - t
    value = 2.0 * rows_n * cols_n * k / dt / 1e12
    desc = (f"oracle (plain C, OpenMP) on {rows_n} rows x {cols_n} cols of C "
            f"(= {rows_n * cols_n} of {m * n} outputs, full k={k}); TFLOP/s on that sample")
    return value, dt, desc, (rows, cols, Cs)


def cpu_phase_breakdown(A, B, k, s, rows, cols):
    """The oracle's phases on the same sample, timed separately (the paper's Fig. 9 split,
    P:613-620): slicing of the sampled rows of A and columns of B, the s(s+1)/2 INT32 pair
    products, and the whole call minus those (accumulation + scaling)."""
    import oracle as O
    As, Bs = np.asfortranarray(A[rows]), np.asfortranarray(B[:, cols])
    rn, cn = len(rows), len(cols)
    t = time.perf_counter()
    da, _, _ = O.split_opA(As, "N", rn, k, rn, s)
    db, _, _ = O.split_opB(Bs, "N", k, cn, k, s)
    t_split = time.perf_counter() - t
    t = time.perf_counter()
    for p in range(1, s + 1):
        for q in range(1, s + 2 - p):
            O.int_gemm(da[p - 1], db[q - 1])
    t_pairs = time.perf_counter() - t
    return {"split_s": t_split, "pair_products_s": t_pairs}


def run_reference(args, wl):
    """--impl reference: the oracle as it stands on the host cores (rank 0 only)."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    if wl.get("complex"):
        print(json.dumps({"impl": "reference", "unavailable": "reference arm times the real "
                          "workloads (C3/C4); C5 is measured GPU-only"}), flush=True)
        return
    import oracle as O
    cores = os.cpu_count()
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    m, n, k, s = wl["m"], wl["n"], wl["k"], wl["s"]
    A = synth.gen_phi(m, k, wl["phi"], wl["seeds"][0])
    B = synth.gen_phi(k, n, wl["phi"], wl["seeds"][1])
    rng = np.random.default_rng(11)
    # each step: a bounded sample (rows x cols of C) sized for ~4 s of CPU work
    r0 = rng.choice(m, 4, replace=False)
    c0 = rng.choice(n, 32, replace=False)
    t = time.perf_counter()
    O.dgemm("N", "N", 4, 32, k, 1.0, np.asfortranarray(A[r0]), 4, np.asfortranarray(B[:, c0]),
            k, 0.0, np.zeros((4, 32), order="F"), 4, s)
    per = max(time.perf_counter() - t, 1e-3) / (4 * 32)
    cols_n = int(min(n, max(32, 4.0 / per / 16)))
    rows_n = 16
    times = []
    for it in range(args.warmup + args.steps):
        rows = np.sort(rng.choice(m, rows_n, replace=False))
        cols = np.sort(rng.choice(n, cols_n, replace=False))
        As, Bs = np.asfortranarray(A[rows]), np.asfortranarray(B[:, cols])
        t = time.perf_counter()
        O.dgemm("N", "N", rows_n, cols_n, k, 1.0, As, rows_n, Bs, k, 0.0,
                np.zeros((rows_n, cols_n), order="F"), rows_n, s)
        dt = time.perf_counter() - t
        if it >= args.warmup:
            times.append(dt)
    sec = float(np.mean(times))
    value = 2.0 * rows_n * cols_n * k / sec / 1e12
    sample = (f"per step: oracle on {rows_n} rows x {cols_n} cols of C (full k={k}), random "
              f"each step; TFLOP/s = 2*rows*cols*k/t")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "i8", "data": "synthetic",
            "config": {"workload": wl["desc"], "m": m, "n": n, "k": k, "s": s, "phi": wl["phi"],
                       "parallelism": "cpu oracle, OpenMP"},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores,
                             "kind": "oracle", "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_zgemm(args, wl):
    """Single-GPU ZGEMM throughput (8mnk/t) vs cuBLAS ZGEMM on the config-5 shape."""
    import torch

    import paper_2306_11975_b200 as oz
    m, n, k, s = wl["m"], wl["n"], wl["k"], wl["s"]
    batch = wl.get("batch", 1)
    torch.cuda.set_device(0)
    psi = synth.gen_phi_complex(m * batch, k, wl["phi"], wl["seeds"][0])
    psi /= np.linalg.norm(psi)
    U = synth.haar_unitary(k, wl["seeds"][1])
    if batch > 1:  # state as (2^(N-d-o), 2^d, 2^o): item b = 2^o x 2^d block, column-major
        dA = torch.from_numpy(np.ascontiguousarray(psi.ravel(order="C"))).cuda()
        dB = torch.from_numpy(np.ascontiguousarray(U.ravel(order="C"))).cuda()  # = U^T col-major
    else:
        dA = torch.from_numpy(np.ascontiguousarray(psi.ravel(order="F"))).cuda()
        dB = torch.from_numpy(np.ascontiguousarray(U.ravel(order="F"))).cuda()
    del psi
    dC = torch.empty(m * n * batch, dtype=torch.complex128, device="cuda")
    h = oz.Handle(0)
    stream = torch.cuda.current_stream()
    h.set_stream(stream)

    def step():
        if batch > 1:  # C_b = A_b U^T: A_b 2^o x 2^d (ld 2^o), shared op(B) = U^T
            h.zgemm_strided_batched("N", "N", m, n, k, 1.0, dA, m, m * k, dB, k, 0, 0.0, dC, m,
                                    m * n, batch, s)
        else:
            h.zgemm("N", "T", m, n, k, 1.0, dA, m, dB, n, 0.0, dC, m, s)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    rep = h.report()
    h.timing_enable(args.steps + 1)
    clocks = ClockSampler(0)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    phases = h.timing_read(args.steps + 1)
    flops = 8.0 * m * n * k * batch
    value = flops / (ms / 1e3) / 1e12
    gemm_ms = float(np.mean([p["gemm_ms"] for p in phases]))
    peaks, src = load_peaks()
    int8_peak = 2.0 * peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    ops = float(s * (s + 1)) * m * batch * (2 * n) * (2 * k)
    achieved = ops / (gemm_ms / 1e3) / 1e12
    if batch > 1:  # torch: out = U @ X, X = state as (batch, 2^d, 2^o) row-major (bmm)
        Um = dB.view(k, n)
        Xm = dA.view(batch, k, m)
        Cm = torch.empty(batch, n, m, dtype=torch.complex128, device="cuda")
        cub = lambda: torch.matmul(Um, Xm, out=Cm)  # noqa: E731
    else:
        Am = dA.view(k, m).t()
        Bm = dB.view(k, n)  # U stored column-major = U^T row-major; op(B) = U^T
        Cm = torch.empty(m, n, dtype=torch.complex128, device="cuda")
        cub = lambda: torch.matmul(Am, Bm, out=Cm)  # noqa: E731
    for _ in range(2):
        cub()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(max(3, args.steps // 2)):
        cub()
    e1.record(stream)
    torch.cuda.synchronize()
    cms = e0.elapsed_time(e1) / max(3, args.steps // 2)
    cv = flops / (cms / 1e3) / 1e12
    line = {"metric": "effective ZGEMM TFLOP/s (8mnk/t) vs cuBLAS ZGEMM", "value": value,
            "unit": "TFLOP/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "i8", "data": "synthetic",
            "config": {"workload": wl["desc"], "m": m, "n": n, "k": k, "s": s,
                       "parallelism": "single GPU", "l2": "inputs larger than L2",
                       "plan": {kk: rep[kk] for kk in ("tile_n", "k_block", "stages",
                                                      "k_chunks", "acc_regions")}},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": int8_peak,
                         "unit": "TFLOP/s", "frac": achieved / int8_peak, "traffic": None,
                         "gemm_ms": gemm_ms, "peak_source": src},
            "cublas_zgemm": {"value": cv, "unit": "TFLOP/s", "ms_per_step": cms,
                             "speedup_ozimmu_vs_cublas": value / cv,
                             "call": "torch.matmul complex128 (cuBLAS ZGEMM%s)" %
                                     (" strided-batched, shared U" if batch > 1 else "")},
            "clocks": clk, "gpu_launches": rep["launches"] * args.steps}
    print(json.dumps(line), flush=True)
    h.close()


def self_launch(args):
    """`bench.py --gpus N` without torchrun: start N ranks (one per GPU) with
    torch.distributed.run on 127.0.0.1 and return its exit code; refuse loudly if fewer than N
    GPUs are visible (OZIMMU_BENCH_ONE_DEVICE=1: the one-GPU test hook, all ranks on cuda:0)."""
    import torch
    ndev = torch.cuda.device_count()
    if os.environ.get("OZIMMU_BENCH_ONE_DEVICE") != "1" and ndev < args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but only {ndev} CUDA device(s) are "
                         "visible; refusing to report a multi-GPU number from fewer GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--local-addr", "127.0.0.1",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--slices", type=int, default=None,
                    help="fixed s; 0 = INT8-AUTO with --auto-T (P:656-659)")
    ap.add_argument("--auto-rule", default="acc", choices=["acc", "loss"],
                    help="INT8-AUTO rule for --slices 0: acc = accuracy-targeted (reading A18, "
                         "default), loss = the paper's mean-mantissa-loss rule (reading A17)")
    ap.add_argument("--auto-T", type=float, default=0.0)
    ap.add_argument("--auto-tau", type=float, default=1.0)
    ap.add_argument("--chunk-cols", type=int, default=0,
                    help="N > 1: columns per broadcast chunk (0 = the library's default, ~n/8)")
    ap.add_argument("--bcast-fp64", action="store_true",
                    help="N > 1: broadcast FP64 B and slice it on every rank (SURVEY s8e byte "
                         "trade-off) instead of B's INT8 planes")
    ap.add_argument("--grid", default=None,
                    help="PRxPC: 2-D partition of C over the N ranks (SURVEY s8e 'large n'); "
                         "default: row blocks")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cublas", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    wl = dict(WORKLOADS[args.config])
    if args.slices is not None:
        wl["s"] = args.slices
    if args.impl == "reference":
        run_reference(args, wl)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if wl.get("complex"):
        run_zgemm(args, wl)
        return

    import torch
    import torch.distributed as dist

    import paper_2306_11975_b200 as oz
    from paper_2306_11975_b200 import dist as D

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    # test hook (never set by the driver): OZIMMU_BENCH_ONE_DEVICE=1 maps every rank to cuda:0
    # and broadcasts over gloo (NCCL refuses two ranks on one GPU), so the N > 1 code path can
    # run on a one-GPU box (timings meaningless: the ranks share one GPU)
    one_dev = os.environ.get("OZIMMU_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # torch.distributed (gloo) is only the bootstrap: the NCCL unique id, barriers and the
        # max-over-ranks of the timings.  The broadcast itself is libozimmu's NCCL communicator.
        dist.init_process_group("gloo")
    dev = torch.device("cuda", local)
    m, n, k, s = wl["m"], wl["n"], wl["k"], wl["s"]
    if world > 1 and s == 0:
        raise SystemExit("bench.py: INT8-AUTO (--slices 0) is single-GPU only (choosing s would "
                         "need A's statistics from every rank)")
    s_call = s  # 0 = INT8-AUTO: every step runs the statistics scan
    pr, pc = world, 1
    if args.grid and world > 1:
        pr, pc = (int(x) for x in args.grid.lower().split("x"))
        assert pr * pc == world, f"--grid {args.grid} needs {pr * pc} ranks, got {world}"
    gi, gj = D.grid_coords(rank, pr, pc)
    r0, r1 = D.row_range(m, pr, gi)
    n0, n1 = D.row_range(n, pc, gj)
    ml, nl = r1 - r0, n1 - n0

    # ---- inputs (identical bytes to the oracle's: synth.gen_phi) ------------------
    A = synth.gen_phi(m, k, wl["phi"], wl["seeds"][0])
    B = synth.gen_phi(k, n, wl["phi"], wl["seeds"][1]) if (rank == 0 or world == 1) else None
    A_loc_h = torch.from_numpy(np.ascontiguousarray(A[r0:r1].ravel(order="F")))
    B_h = torch.from_numpy(B.ravel(order="F")) if B is not None else None
    dA = A_loc_h.to(dev)
    dB = B_h.to(dev) if B_h is not None else None
    dC = torch.empty(max(1, ml * nl), dtype=torch.float64, device=dev)
    lda = max(1, ml)

    h = oz.Handle(local)
    stream = torch.cuda.current_stream(dev)
    h.set_stream(stream)
    if s == 0:
        if args.auto_rule == "loss":
            h.set_auto(args.auto_T, 18)
        else:
            h.set_auto_accuracy(args.auto_tau, 18)
    engine = engines = None
    if world > 1:
        h.set_dist(args.chunk_cols, RESERVE_SMS, args.bcast_fp64)
        if one_dev:
            make = lambda g, mem: D.BcastEngine(h, g, mem)  # noqa: E731
        else:
            def make(g, mem):
                return D.NcclEngine(h, D.make_nccl_comm(local, g, RESERVE_SMS, mem))
        if pc > 1:
            engines = D.make_grid_engines(make, pr, pc, 0)
        else:
            engine = make(None, list(range(world)))

    def step():
        if world == 1:
            h.dgemm("N", "N", m, n, k, 1.0, dA, m, dB, k, 0.0, dC, m, s_call)
        elif engines is not None:
            D.dgemm_grid2d(engines, pr, pc, "N", "N", ml, n, k, 1.0, dA, lda, dB, k, 0.0, dC, lda,
                           s_call, root=0)
        else:
            D.dgemm_rowblock(engine, "N", "N", ml, n, k, 1.0, dA, lda, dB, k, 0.0, dC, lda,
                             s_call, root=0)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    rep = h.report()
    if s == 0:
        wl["auto"] = {"rule": args.auto_rule,
                      ("T" if args.auto_rule == "loss" else "tau"):
                          (args.auto_T if args.auto_rule == "loss" else args.auto_tau),
                      "chosen_s": rep["num_slices"], "capped": bool(rep["auto_capped"])}
        s = rep["num_slices"]  # for the op counts below; every timed step re-runs the scan

    # ---- timed region: inputs resident in HBM -------------------------------------
    h.timing_enable(args.steps + 1)
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    phases = h.timing_read(args.steps + 1)
    h.timing_enable(0)
    if world > 1:  # max over ranks (gloo: CPU tensor)
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    flops = 2.0 * m * n * k
    value = flops / (ms / 1e3) / 1e12
    bcast = None
    if world > 1 and phases:
        # the library marks the end of the last broadcast on its collective stream: start ->
        # last chunk received, and the payload this rank received (INT8 planes + exponents, or
        # FP64 B); SURVEY s8e byte trade-off: s vs 8 bytes per element of op(B)
        k_pad = (k + 15) // 16 * 16
        payload = (8 * k * nl) if (args.bcast_fp64) else (s * nl * k_pad + 4 * nl)
        t_b = float(np.mean([p["slice_b_ms"] for p in phases]))
        bcast = {"payload_bytes_per_rank": int(payload), "ms_start_to_last_chunk": t_b,
                 "gbps_effective": payload / (t_b / 1e3) / 1e9 if t_b > 0 else None,
                 "payload": "fp64 op(B)" if args.bcast_fp64 else "INT8 planes + exponents",
                 "chunk_cols": args.chunk_cols or "library default (~n/8)",
                 "reserve_sms": RESERVE_SMS, "nccl_max_ctas": RESERVE_SMS,
                 "transport": "gloo host-staged (one-device test hook)" if one_dev
                 else "NCCL (libozimmu's communicator)"}

    # ---- dominant kernel: the fused GEMM (per-launch CUDA events on our stream) --------
    gemm_ms = float(np.mean([p["gemm_ms"] for p in phases])) if phases else None
    # A and B are sliced concurrently (two streams): the phase lasts max(start->A, start->B)
    slice_ms = float(np.mean([max(p["slice_a_ms"], p["slice_b_ms"]) for p in phases])) if phases else None
    peaks, peak_src = load_peaks()
    int8_peak = 2.0 * peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    # N = 1: one GEMM launch per call; N > 1: gemm_ms spans this rank's GEMM launches of a
    # call (1, 1, 2, 4, .. column chunks each), so the ops are all of the rank's block
    n_launch = n if world == 1 else nl
    int8_ops_launch = float(s * (s + 1)) * ml * n_launch * k  # 2 ops per INT8 MAC
    achieved = int8_ops_launch / (gemm_ms / 1e3) / 1e12 if gemm_ms else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_gemm_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pj = json.load(f)
            if pj.get("workload") == args.config and pj.get("s") == s and world == 1:
                traffic = pj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    int8_burst = 2.0 * peaks.get("bf16_tflops", int8_peak / 2.0)
    hw_at_clock = None
    if clk.get("sm_mhz"):
        hw_at_clock = 148 * 8192 * 2 * clk["sm_mhz"] * 1e6 / 1e12  # INT8 MAC/clk/SM x 2 ops
    s_run = rep.get("num_slices") or s  # the s the library ran (INT8-AUTO: its choice)
    slice_bytes = (8 + s_run) * (ml * k + k * n) + 4 * (ml + n)
    roofline = {"bound": "tensor", "kernel": "k_oz_gemm (tcgen05.mma.kind::i8 + FP64 epilogue)",
                "achieved": achieved, "peak": int8_peak, "unit": "TFLOP/s",
                "frac": (achieved / int8_peak) if achieved else None, "traffic": traffic,
                "frac_of_burst_peak": (achieved / int8_burst) if achieved else None,
                "tensor_util_at_measured_clock": (achieved / hw_at_clock)
                if (achieved and hw_at_clock) else None,
                "ops_per_launch": int8_ops_launch,
                "ops": "INT8 ops (2 per MAC) = s(s+1) m_loc n_loc k over the GEMM span of a call "
                       "(one launch at N = 1)",
                "peak_source": f"{peak_src} MEASURED_PEAKS.json; {INT8_PEAK_NOTE}",
                "gemm_ms": gemm_ms, "slice_ms": slice_ms,
                "gemm_share_of_step": (gemm_ms / ms) if gemm_ms else None,
                # the GEMM runs at the board power cap: INT8 work per joule is its real limit
                "int8_tops_per_watt": (achieved / clk["power_w_median"])
                if (achieved and clk.get("power_w_median")) else None,
                "effective_fp64_gflops_per_watt": (value * 1e3 / clk["power_w_median"])
                if clk.get("power_w_median") else None,
                "library_context": library_int8_context(),
                # the slicing phase (A2 + A3): op(A) and op(B) sliced concurrently, HBM-bound;
                # algorithmic bytes = 8 read + s written per element + 4 per vector, and at N = 1
                # the strided op(A) of this workload reads A once more for its exponent scan
                "slicing": ({"bound": "hbm", "ms": slice_ms, "s": s_run,
                             "algorithmic_bytes": slice_bytes,
                             "achieved_GBps": slice_bytes / (slice_ms * 1e-3) / 1e9,
                             "peak_GBps": peaks.get("hbm_gbs"),
                             "frac": slice_bytes / (slice_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]
                             if peaks.get("hbm_gbs") else None}
                            if (slice_ms and world == 1) else None)}

    # ---- cuBLAS DGEMM on the same GPUs (row block, B resident: no communication) -----
    cublas = None
    if not args.no_cublas:
        # non-root ranks regenerate B (same seed) instead of receiving it: no communication
        Bt = dB if dB is not None else torch.from_numpy(
            synth.gen_phi(k, n, wl["phi"], wl["seeds"][1]).ravel(order="F")).to(dev)
        Am = dA.view(k, ml).t() if ml else None
        Bm = Bt.view(n, k).t()[:, n0:n1]
        Cm = torch.empty(ml, nl, dtype=torch.float64, device=dev)

        def cstep():
            if ml:
                torch.matmul(Am, Bm, out=Cm)
        for _ in range(2):
            cstep()
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(max(3, args.steps // 2)):
            cstep()
        e1.record(stream)
        torch.cuda.synchronize()
        cms = e0.elapsed_time(e1) / max(3, args.steps // 2)
        if world > 1:
            t = torch.tensor([cms], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            cms = float(t.item())
        cv = flops / (cms / 1e3) / 1e12
        cublas = {"value": cv, "unit": "TFLOP/s", "ms_per_step": cms,
                  "frac_of_fp64_peak_40": cv / 40.0 / world, "speedup_ozimmu_vs_cublas": value / cv,
                  "note": "torch.matmul float64 (cuBLAS DGEMM), same C blocks, B already resident"}
        if world > 1 or args.no_cpu_baseline:
            del Cm
        if world > 1:
            del Bt

    # ---- e2e: public API with HOST buffers (pinned), copies inside the timed region ---
    e2e = None
    if not args.no_e2e:
        A_pin = A_loc_h.pin_memory()
        B_pin = B_h.pin_memory() if B_h is not None else None
        C_pin = torch.empty(ml * nl, dtype=torch.float64).pin_memory()
        h2d = A_pin.numel() * 8 + (B_pin.numel() * 8 if B_pin is not None else 0)
        d2h = C_pin.numel() * 8

        def estep():
            if world == 1:  # the host-buffer C-ABI call: copies overlapped inside the library
                h.dgemm_host("N", "N", m, n, k, 1.0, A_pin, m, B_pin, k, 0.0, C_pin, m, s_call)
                return
            dA.copy_(A_pin, non_blocking=True)
            if B_pin is not None:
                dB.copy_(B_pin, non_blocking=True)
            step()
            C_pin.copy_(dC, non_blocking=True)
        estep()
        torch.cuda.synchronize()
        esteps = max(3, min(args.steps, 5))
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(esteps):
            estep()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        wall = (time.perf_counter() - t0) / esteps * 1e3
        ems = e0.elapsed_time(e1) / esteps
        if world > 1:
            t = torch.tensor([ems, wall], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems, wall = float(t[0].item()), float(t[1].item())
        same = None
        if world == 1:  # the host-buffer result equals the device-pointer result bit for bit
            step()
            torch.cuda.synchronize()
            same = bool(torch.equal(C_pin, dC.cpu()))
        e2e = {"value": flops / (ems / 1e3) / 1e12, "unit": "TFLOP/s",
               "bitexact_vs_device_call": same,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": ems, "wall_ms_per_step": wall, "steps": esteps,
               "note": ("ozimmu_dgemm_host on pinned-host A, B -> C (A row blocks and B column "
                        "chunks transferred alternately, each followed by one GEMM over the newly "
                        "computable C region, whose D2H starts as soon as it is done; H2D, "
                        "slicing, GEMM and D2H overlap on 3 streams; blocks until C is in host "
                        "memory)") if world == 1 else
                       "ozimmu_dgemm on pinned-host A,B -> C via cudaMemcpyAsync on the same "
                       "stream (rank-local bytes; root also copies B)"}

    # ---- CPU baseline (oracle) + accuracy on the same sample (rank 0, N = 1) ------------
    cpu = None
    accuracy = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
        # the GPU result of the last timed step
        step()
        torch.cuda.synchronize()
        cv_, dt_, desc, (rows, cols, Cs) = cpu_baseline_sample(A, B, k, s)
        cpu = {"value": cv_, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "oracle",
               "sample": desc, "seconds": dt_, "cpu_model": cpu_model()}
        ph = cpu_phase_breakdown(A, B, k, s, rows, cols)
        ph["accumulate_s"] = max(0.0, dt_ - ph["split_s"] - ph["pair_products_s"])
        ph["note"] = ("oracle phases on the same sample (P:613-620 Fig. 9 split): accumulate = "
                      "whole call - split - pair products")
        cpu["phases"] = ph
        Cg = dC.view(n, m).t()[torch.as_tensor(rows, device=dev)][:, torch.as_tensor(cols, device=dev)]
        Cg = Cg.cpu().numpy()
        import oracle as O
        hi, lo = O.dd_gemm("N", "N", len(rows), len(cols), k, np.asfortranarray(A[rows]),
                           len(rows), np.asfortranarray(B[:, cols]), k)
        st = O.err_stats(Cg, hi, lo)
        # condition of each sampled output, (|A||B|)_ij / |C_ij| (the literal max_rel is driven
        # by huge ones); the diagnostic restricts max_rel to cond <= 4 x median
        absAB = np.abs(A[rows]) @ np.abs(B[:, cols])
        cond = absAB / np.maximum(np.abs(hi), np.finfo(float).tiny)
        well = cond <= 4.0 * np.median(cond)
        ref_abs = np.abs(hi)

        def cond_max_rel(Cx):
            d = np.abs((Cx - hi) - lo)
            sel = well & (ref_abs > 0)
            return float((d[sel] / ref_abs[sel]).max()) if sel.any() else None
        accuracy = {"vs": "double-double (oracle/dd_ref.c) on the cpu_baseline sample",
                    "max_rel": st["max_rel"], "mean_rel": st["mean_rel"], "nw_max": st["nw_max"],
                    "max_rel_cond_le_4x_median": cond_max_rel(Cg),
                    "cond_median": float(np.median(cond)), "cond_max": float(cond.max()),
                    "bitexact_vs_oracle": bool(np.array_equal(Cg, Cs))}
        if cublas is not None:  # cuBLAS DGEMM's full-size result on the same sample
            Cc = Cm[torch.as_tensor(rows, device=dev)][:, torch.as_tensor(cols, device=dev)]
            Cc = Cc.cpu().numpy()
            sc = O.err_stats(Cc, hi, lo)
            accuracy["cublas"] = {"max_rel": sc["max_rel"], "mean_rel": sc["mean_rel"],
                                  "nw_max": sc["nw_max"],
                                  "max_rel_cond_le_4x_median": cond_max_rel(Cc)}
            del Cm
        mr_cub = accuracy.get("cublas", {}).get("mean_rel")
        accuracy["gate"] = ("nw_max <= 1e-14 and mean_rel <= min(1e-14, cuBLAS mean_rel) "
                            "(SURVEY s8c reading A14)")
        accuracy["gate_pass"] = bool(st["nw_max"] <= 1e-14 and st["mean_rel"] <= 1e-14 and
                                     (mr_cub is None or st["mean_rel"] <= mr_cub))

    launches_per_step = rep.get("launches", 0)
    if world > 1:  # rank 0's kernels per step (its slicing of every B chunk included)
        engs = [e for e in (engines or [engine]) if e is not None]
        launches_per_step = sum(e.launches for e in engs)
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "i8", "data": "synthetic",
        "config": {"workload": wl["desc"], "m": m, "n": n, "k": k, "s": s, "phi": wl["phi"],
                   "seeds": list(wl["seeds"]), "auto": wl.get("auto"),
                   "parallelism": "single GPU" if world == 1 else (
                       f"C row blocks x{world} + chunked NCCL broadcast of B slices" if pc == 1
                       else f"C {pr}x{pc} blocks + chunked NCCL broadcast of each column "
                            f"block's B slices within its grid column"),
                   "l2": "inputs larger than L2 (each operand 2.1 GB fp64 + 2.4 GB int8 planes)",
                   "io_dtype": "f64 in/out; i8 x i8 -> i32 tensor-core products; f64 epilogue",
                   "plan": {kk: rep[kk] for kk in ("tile_n", "k_block", "stages", "k_chunks",
                                                  "slice_width")}},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "cublas_dgemm": cublas,
        "accuracy": accuracy,
        "clocks": clk,
        "gpu_launches": int(launches_per_step * args.steps),
        "phases_ms_mean": {"slice": slice_ms, "gemm": gemm_ms},
        "bcast": bcast,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    h.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
