#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py launches <launches.csv>      # per-kernel time shares
    python tools/ncu_summary.py full <report.ncu-rep>        # key metrics of a --set full capture
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    idx = {k: j for j, k in enumerate(hdr)}
    agg = defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        agg[r[idx["Kernel Name"]]].append(float(r[idx["Metric Value"]]))
    tot = sum(sum(v) for v in agg.values())
    print("kernel launches (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)")
    print("%6s %12s %12s %7s  %s" % ("count", "total_us", "avg_us", "share", "kernel"))
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print("%6d %12.1f %12.1f %6.1f%%  %s" % (len(v), sum(v) / 1e3, sum(v) / len(v) / 1e3,
                                                100 * sum(v) / tot, k[:110]))


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print("kernel:", d.get("Kernel Name", "?")[:120])
        for k in KEYS:
            if k in d:
                print("  %-80s %14s %s" % (k, d[k], u.get(k, "")))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
