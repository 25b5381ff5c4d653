#!/usr/bin/env python3
"""Device time of one config's insert and lookup phases under forced
variants (AUTO vs direct vs blocked), L2 flushed before each phase pair.

    python scripts/variant_ab.py <config> [reps]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2101_01719_b200 import SplitBlockFilter, _lib  # noqa: E402
from paper_2101_01719_b200 import workload as W  # noqa: E402

cid = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = W.CONFIGS[cid]
st = W.StreamHandle(cfg.inserts)
N, L = cfg.inserts.n, cfg.lookups.n
ins = W.gen_inserts(st, 0, N)
look = W.gen_lookups(st, cfg.lookups, N, 0, L)
bits = torch.empty((L + 31) // 32, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
chunk = cfg.insert_chunk or N
f = SplitBlockFilter(cfg.num_buckets)
for _ in range(3):  # untimed warm-up: clocks, pool growth, plan
    f.clear()
    for s in range(0, N, chunk):
        f.add_hashes(ins[s:s + chunk])
    f.find_hashes_bits(look, bits)
torch.cuda.synchronize()
for iv, fv, name in [(0, 0, "auto"), (0, _lib.FIND_SMEM, "smem"), (_lib.INSERT_WIDE_TEST, _lib.FIND_GLOBAL, "direct"),
                     (_lib.INSERT_BLOCKED, _lib.FIND_BLOCKED, "blocked"), (_lib.INSERT_WIDE, _lib.FIND_GLOBAL, "wide")]:
    try:
        f.set_insert_variant(iv)
        f.set_find_variant(fv)
    except Exception as exc:  # e.g. SMEM on a filter too large for shared memory
        print(f"cfg{cid} {name:8s} skipped: {exc}")
        continue
    ti, tl = [], []
    for r in range(reps + 1):
        f.clear()
        flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        for s in range(0, N, chunk):
            f.add_hashes(ins[s:s + chunk])
        e[1].record()
        f.find_hashes_bits(look, bits)
        e[2].record()
        torch.cuda.synchronize()
        if r:
            ti.append(e[0].elapsed_time(e[1]))
            tl.append(e[1].elapsed_time(e[2]))
    mi, ml = statistics.mean(ti), statistics.mean(tl)
    print(f"cfg{cid} {name:8s} insert {mi:8.3f} ms {N / mi / 1e6:7.1f} G/s   lookup {ml:8.3f} ms {L / ml / 1e6:7.1f} G/s  "
          f"crc-probe {int(bits[:1000].sum())}")
