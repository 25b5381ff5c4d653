#!/usr/bin/env python3
"""One full phase (insert or lookup) of a BASELINE config under the CUDA
profiler range, for ncu launch lists per phase (`ncu --profile-from-start off`).

    python scripts/profile_phase.py <config> <insert|lookup>

Inputs are generated and (for lookups) the filter built outside the range;
inside it runs exactly what bench.py times for that phase (AUTO variants,
the config's insert chunks, bitmap lookups)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2101_01719_b200 import SplitBlockFilter  # noqa: E402
from paper_2101_01719_b200 import workload as W  # noqa: E402

cid, phase = int(sys.argv[1]), sys.argv[2]
cfg = W.CONFIGS[cid]
st = W.StreamHandle(cfg.inserts)
N, L = cfg.inserts.n, cfg.lookups.n
chunk = cfg.insert_chunk or N
ins = W.gen_inserts(st, 0, N)
f = SplitBlockFilter(cfg.num_buckets)


def insert_all():
    for s in range(0, N, chunk):
        f.add_hashes(ins[s:s + chunk])


if phase == "insert":
    insert_all()                      # warm-up (plans, pool) outside the range
    f.clear()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    insert_all()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
else:
    insert_all()
    look = W.gen_lookups(st, cfg.lookups, N, 0, L)
    bits = torch.empty((L + 31) // 32, dtype=torch.int32, device="cuda")
    f.find_hashes_bits(look, bits)    # warm-up outside the range
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    f.find_hashes_bits(look, bits)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
print("done", cid, phase)
