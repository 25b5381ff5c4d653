#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (run here, no GPU needed).

    python scripts/summarize_ncu.py report <x.ncu-rep> [--keys N] [--bytes-per-key B]
    python scripts/summarize_ncu.py launches <launches.csv>
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_requests_srcunit_tex_op_red.sum",
    "lts__t_sectors_srcunit_tex_op_red.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard", "dram__sectors_read.sum",
]


def report(path: str, keys: int | None, bpk: float | None) -> str:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = [f"### {path.split('/')[-1]}", ""]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")]
        lines.append(f"kernel: `{name}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        got = {}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                lines.append(f"| {m} | {vals[i]} | {units[i]} |")
                got[m] = (vals[i], units[i])
        if keys:
            def tobytes(v, u):
                v = float(v.replace(",", ""))
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            rd = tobytes(*got["dram__bytes_read.sum"])
            wr = tobytes(*got["dram__bytes_write.sum"])
            lines.append(f"| DRAM bytes / key (read+write) | {(rd + wr) / keys:.2f} | B |")
            if bpk:
                lines.append(f"| algorithmic bytes / key | {bpk} | B |")
        lines.append("")
    return "\n".join(lines)


def launches(path: str) -> str:
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    lines = [f"### launch list {path.split('/')[-1]} (ncu --metrics gpu__time_duration.sum, cold, serialised)",
             "", "| kernel | launches | mean ns | total ns |", "|---|---|---|---|"]
    for k, v in agg.items():
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.0f} | {sum(v):.0f} |")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "report":
        keys = bpk = None
        if "--keys" in sys.argv:
            keys = int(sys.argv[sys.argv.index("--keys") + 1])
        if "--bytes-per-key" in sys.argv:
            bpk = float(sys.argv[sys.argv.index("--bytes-per-key") + 1])
        print(report(sys.argv[2], keys, bpk))
    else:
        print(launches(sys.argv[2]))
