"""Summarise ncu reports (run here, no GPU): launch list shares and key metrics of a
full capture.  usage: python tools/ncu_summary.py launches.csv [prof.ncu-rep ...]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    out = []
    for r in rows[hi + 1:]:
        if len(r) > vi:
            out.append((r[ki].split("(")[0].replace("void ", ""), float(r[vi].replace(",", ""))))
    tot = sum(v for _, v in out)
    agg = {}
    for k, v in out:
        agg.setdefault(k, [0, 0.0])
        agg[k][0] += 1
        agg[k][1] += v
    return {k: {"launches": c, "total_ns": t, "share": t / tot} for k, (c, t) in agg.items()}


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in h:
                d[k] = r[h.index(k)]
        res.append(d)
    return res


if __name__ == "__main__":
    out = {}
    for p in sys.argv[1:]:
        out[p] = launches(p) if p.endswith(".csv") else full(p)
    print(json.dumps(out, indent=1))
