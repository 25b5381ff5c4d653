#!/usr/bin/env python3
"""Print an ncu --csv --metrics launch list as one line per launch."""
import csv
import sys

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    launches = {}
    for r in rows[1:]:
        launches.setdefault(r[ii], {"k": r[ki].split("(")[0][-34:]})[r[mi]] = (r[vi], r[ui])
    print("==", path)
    for v in list(launches.values())[-int(sys.argv[0] and 14):]:
        t = v.get("gpu__time_duration.sum", ("", ""))
        rd = v.get("dram__bytes_read.sum", ("", ""))
        wr = v.get("dram__bytes_write.sum", ("", ""))
        hit = v.get("lts__t_sector_hit_rate.pct", ("", ""))
        print(f"  {v['k']:34s} t={t[0]:>10s}{t[1]:3s} rd={rd[0]:>14s}{rd[1]:6s} wr={wr[0]:>14s}{wr[1]:6s} hit={hit[0]}")
