#!/usr/bin/env python3
"""Summarise per-phase ncu launch lists into profiles/traffic.json.

    python scripts/traffic.py <tag> <cid>:<phase>:<launches.csv> ...

For each (config, phase): the sum over every kernel the phase launched of
dram__bytes_read.sum + dram__bytes_write.sum and gpu__time_duration.sum
(cold, serialised replays), per key of the phase (inserts or lookups)."""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2101_01719_b200 import workload as W  # noqa: E402

SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TS = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1, "s": 1}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    L = collections.OrderedDict()
    for r in rows[1:]:
        d = L.setdefault(r[ii], {"kernel": r[ki].split("(")[0]})
        d[r[mi]] = float(r[vi].replace(",", "")) * (SC.get(r[ui], 1) if "bytes" in r[mi] else TS.get(r[ui], 1))
    return list(L.values())


def main():
    tag = sys.argv[1]
    path = os.path.join(ROOT, "profiles", "traffic.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    out["_note"] = ("DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) summed over every kernel of one "
                    "phase of a BASELINE config (scripts/profile_phase.py under ncu --profile-from-start off, "
                    "--clock-control none: cold, serialised launches), per key of that phase. bench.py scales "
                    "the per-key figure to the run's keys as roofline.traffic / insert_roofline.traffic.")
    for spec in sys.argv[2:]:
        cid, phase, csvp = spec.split(":", 2)
        cfg = W.CONFIGS[int(cid)]
        keys = cfg.inserts.n if phase == "insert" else cfg.lookups.n
        ls = launches(csvp)
        rd = sum(d.get("dram__bytes_read.sum", 0) for d in ls)
        wr = sum(d.get("dram__bytes_write.sum", 0) for d in ls)
        t = sum(d.get("gpu__time_duration.sum", 0) for d in ls)
        per = collections.Counter()
        for d in ls:
            per[d["kernel"].replace("void ", "").split("::")[-1]] += 1
        out.setdefault(cid, {})[phase] = {
            "keys": keys, "launches": len(ls), "kernels": dict(per),
            "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes_per_key": (rd + wr) / keys,
            "ncu_time_s": t, "source": f"profiles/{tag}_launch_{cid}_{phase}.csv"}
        print(f"config {cid} {phase}: {len(ls)} launches, {(rd + wr) / keys:.2f} B/key DRAM, {t * 1e3:.2f} ms (ncu)")
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
