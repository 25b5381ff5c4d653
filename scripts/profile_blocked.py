#!/usr/bin/env python3
"""Run one path on one config a few times (for ncu launch lists / captures).

    python scripts/profile_blocked.py <config> <insert|find> <variant> [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2101_01719_b200 import SplitBlockFilter  # noqa: E402
from paper_2101_01719_b200 import workload as W  # noqa: E402

cid, op, variant = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cfg = W.CONFIGS[cid]
st = W.StreamHandle(cfg.inserts)
N = cfg.inserts.n
L = min(cfg.lookups.n, 1 << 28)
f = SplitBlockFilter(cfg.num_buckets)
chunk = cfg.insert_chunk or N
ins = W.gen_inserts(st, 0, min(N, 1 << 28))
if op == "insert":
    f.set_insert_variant(variant)
    for _ in range(reps):
        f.clear()
        for s in range(0, ins.numel(), chunk):
            f.add_hashes(ins[s:s + chunk])
else:
    for s in range(0, ins.numel(), chunk):
        f.add_hashes(ins[s:s + chunk])
    look = W.gen_lookups(st, cfg.lookups, N, 0, L)
    bits = torch.empty((L + 31) // 32, dtype=torch.int32, device="cuda")
    f.set_find_variant(variant)
    for _ in range(reps):
        f.find_hashes_bits(look, bits)
torch.cuda.synchronize()
print("done", cid, op, variant)
