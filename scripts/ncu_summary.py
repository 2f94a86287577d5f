#!/usr/bin/env python
"""Summarise ncu output brought back in gpurun_out/ into text files under profiles/.

    python scripts/ncu_summary.py launches gpurun_out/launches.csv  > profiles/<name>.txt
    python scripts/ncu_summary.py report   gpurun_out/prof_x.ncu-rep [alg_bytes] [alg_flops] > profiles/<name>.txt

`launches` aggregates a --metrics gpu__time_duration.sum launch list per kernel
(count, total, mean, share).  `report` prints the headline metrics of a
--set full capture, DRAM traffic against the algorithmic bytes (or tensor-pipe
activity against the algorithmic FLOPs), and the warp-stall breakdown.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3}.get(d.get("Metric Unit", "ns"), 1e-3)
        k = d["Kernel Name"]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':110s} {'n':>4s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:110]:110s} {n:4d} {t:10.1f} {t / n:9.1f} {100 * t / tot:5.1f}%")


HEAD = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
]


def report(path, alg_bytes=None, alg_flops=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        print(f"Kernel Name  {d.get('Kernel Name', '?')}")
        for k in HEAD:
            if k in d:
                print(f"  {k:64s} {d[k]:>16s} {u.get(k, '')}")
        def val(k, to_bytes=False):
            v = float(d[k].replace(",", ""))
            if to_bytes:
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.get(k, "byte"), 1)
            return v
        t_us = val("gpu__time_duration.sum") * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(
            u.get("gpu__time_duration.sum", "usecond"), 1.0)
        traffic = val("dram__bytes_read.sum", True) + val("dram__bytes_write.sum", True)
        print(f"  dram traffic (read+write) per launch: {traffic:.0f} B")
        if alg_bytes:
            print(f"  algorithmic bytes per launch:         {alg_bytes:.0f} B  (traffic = {100 * traffic / alg_bytes:.1f}%)")
            print(f"  achieved (algorithmic / ncu duration {t_us:.2f} us, cold, serialised): "
                  f"{alg_bytes / t_us / 1e3:.0f} GB/s")
        if alg_flops:
            print(f"  algorithmic FLOPs per launch: {alg_flops:.4g}; achieved {alg_flops / t_us / 1e6:.1f} TFLOP/s"
                  f" (ncu duration {t_us:.1f} us)")
        stalls = {k: val(k) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
        tot = sum(stalls.values())
        if tot:
            print("  warp stall samples:")
            for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:12]:
                print(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {v:10.0f} {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        ab = float(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "-" else None
        af = float(sys.argv[4]) if len(sys.argv) > 4 else None
        report(sys.argv[2], ab, af)
