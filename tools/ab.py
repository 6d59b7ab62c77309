"""A/B timing of library variants (development tool).

    python tools/ab.py N s lib1.so lib2.so ... [--rounds R] [--trans NN] [--iters I]

Each variant runs in its own subprocess (OZIMMU_LIB=..., "default" = the product library),
on the same seeded phi = 0.5 inputs: 3 warm-up calls, then `iters` CUDA-event-timed calls
back to back; prints median ms, effective TFLOP/s, median SM clock / power during the timed
calls and a hash of C (variants must agree bitwise).  Rounds alternate the variants to
expose power/clock drift.
"""
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(N, s, iters, trans):
    sys.path.insert(0, ROOT)
    import torch
    import paper_2306_11975_b200 as oz
    g = torch.Generator(device="cuda").manual_seed(1)

    def gen():
        u = torch.rand(N, N, dtype=torch.float64, device="cuda", generator=g) - 0.5
        return u * torch.exp(0.5 * torch.randn(N, N, dtype=torch.float64, device="cuda", generator=g))
    A, B = gen(), gen()
    C = torch.empty(N, N, dtype=torch.float64, device="cuda")
    h = oz.Handle(0)

    def f():
        h.dgemm(trans[0], trans[1], N, N, N, 1.0, A, N, B, N, 0.0, C, N, s)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    samples = []
    stop = threading.Event()

    def sampler():
        while not stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                                      "--format=csv,noheader,nounits", "-i", "0"],
                                     capture_output=True, text=True, timeout=5).stdout
                a, b = out.strip().split(",")
                samples.append((float(a), float(b)))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.2)
    th = threading.Thread(target=sampler, daemon=True)
    th.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(iters)]
    for e0, e1 in ev:
        e0.record()
        f()
        e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ts = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
    ms = ts[len(ts) // 2]
    clk = sorted(x[0] for x in samples)
    pw = sorted(x[1] for x in samples)
    hsh = hashlib.sha1(C.cpu().numpy().tobytes()).hexdigest()[:12]
    print(json.dumps({"lib": os.path.basename(os.environ.get("OZIMMU_LIB", "default")),
                      "env": os.environ.get("AB_TAG", ""), "N": N,
                      "s": s, "ms": round(ms, 3), "tflops": round(2.0 * N ** 3 / ms / 1e9, 2),
                      "min_ms": round(ts[0], 3), "max_ms": round(ts[-1], 3),
                      "sm_mhz": clk[len(clk) // 2] if clk else None,
                      "power_w": pw[len(pw) // 2] if pw else None, "hash": hsh}), flush=True)


def main():
    if sys.argv[1] == "--child":
        child(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5])
        return
    args = sys.argv[1:]
    opts = {"--rounds": "2", "--trans": "NN", "--iters": "8"}
    for k in list(opts):
        if k in args:
            i = args.index(k)
            opts[k] = args[i + 1]
            del args[i:i + 2]
    N, s, libs = int(args[0]), int(args[1]), args[2:]
    for _ in range(int(opts["--rounds"])):
        for lib in libs:
            env = dict(os.environ)
            # "lib@VAR=val,VAR2=val" runs the variant with extra environment
            lib, _, extra = lib.partition("@")
            for kv in filter(None, extra.split(",")):
                k, _, v = kv.partition("=")
                env[k] = v
            if lib != "default":
                env["OZIMMU_LIB"] = os.path.abspath(lib)
            env["AB_TAG"] = extra
            subprocess.run([sys.executable, __file__, "--child", str(N), str(s), opts["--iters"],
                            opts["--trans"]], env=env, check=False)


if __name__ == "__main__":
    main()
