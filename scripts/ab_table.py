#!/usr/bin/env python3
"""Table of bench.py A/B lines: python scripts/ab_table.py gpurun_out/<prefix>*.json"""
import json
import sys

for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001
        print(f"{p}: unreadable ({exc})")
        continue
    print(f"{p.split('/')[-1]:28s} step {d.get('value', 0):7.2f}  ins {d.get('insert_gkeys_s', 0):7.2f}  "
          f"look {d.get('lookup_gkeys_s', 0):7.2f}  max/min {d.get('step_max_over_min', 0):.3f}  "
          f"parity {d.get('parity', {}).get('matches_reference')}")
