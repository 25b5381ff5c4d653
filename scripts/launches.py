#!/usr/bin/env python3
"""One line per launch of an ncu --csv --metrics launch list: time, DRAM bytes, L2 hit rate.

    python scripts/launches.py <launches.csv> [last_n] [keys_for_bytes_per_key]
"""
import collections
import csv
import sys

path = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 12
keys = float(sys.argv[3]) if len(sys.argv) > 3 else 0
rows = [r for r in csv.reader(open(path)) if len(r) > 5]
hdr = rows[0]
ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
L = collections.OrderedDict()
for r in rows[1:]:
    d = L.setdefault(r[ii], {"k": r[ki].split("(")[0][-44:]})
    v = r[vi].replace(",", "")
    try:
        v = float(v)
    except ValueError:
        pass
    d[r[mi]] = (v, r[ui])
SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TS = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1, "ms": 1, "second": 1e3}
for d in list(L.values())[-last:]:
    t = d["gpu__time_duration.sum"]
    ms = t[0] * TS.get(t[1], 1)
    rd = d.get("dram__bytes_read.sum", (0, "byte"))
    wr = d.get("dram__bytes_write.sum", (0, "byte"))
    rdb, wrb = rd[0] * SC.get(rd[1], 1), wr[0] * SC.get(wr[1], 1)
    hit = d.get("lts__t_sector_hit_rate.pct", ("", ""))[0]
    extra = f" ({rdb / keys:.2f} + {wrb / keys:.2f} B/key)" if keys else ""
    print(f"  {d['k']:44s} {ms:8.3f} ms  rd {rdb / 1e9:7.3f} GB  wr {wrb / 1e9:7.3f} GB{extra}  L2 hit {hit}")
