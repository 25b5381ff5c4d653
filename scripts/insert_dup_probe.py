#!/usr/bin/env python3
"""Config-4 insert phase with and without its Zipf duplicates: 15 x 2^26-key
calls into a fresh 1 GiB filter, device-timed (L2 flushed before each rep).

    python scripts/insert_dup_probe.py [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2101_01719_b200 import SplitBlockFilter  # noqa: E402
from paper_2101_01719_b200 import workload as W  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = W.CONFIGS[4]
N, chunk = cfg.inserts.n, cfg.insert_chunk
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, spec in [("zipf", cfg.inserts), ("distinct", W.InsertSpec(seed=7, n=N))]:
    ins = W.gen_inserts(W.StreamHandle(spec), 0, N)
    f = SplitBlockFilter(cfg.num_buckets)
    ts = []
    for r in range(reps + 2):
        f.clear()
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in range(0, N, chunk):
            f.add_hashes(ins[s:s + chunk])
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    ms = sum(ts) / len(ts)
    print(f"{name:9s} insert phase {ms:8.3f} ms  {N / ms / 1e6:6.1f} Gkeys/s")
    del ins, f
