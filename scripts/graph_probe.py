#!/usr/bin/env python3
"""Does replaying the config-2 step (insert + lookup) as a CUDA graph change
the device time? (launch latency vs the 64 us step)"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2101_01719_b200 import SplitBlockFilter  # noqa: E402
from paper_2101_01719_b200 import workload as W  # noqa: E402

cfg = W.CONFIGS[2]
st = W.StreamHandle(cfg.inserts)
ins = W.gen_inserts(st, 0, cfg.inserts.n)
look = W.gen_lookups(st, cfg.lookups, cfg.inserts.n, 0, cfg.lookups.n)
bits = torch.empty((cfg.lookups.n + 31) // 32, dtype=torch.int32, device="cuda")
f = SplitBlockFilter(cfg.num_buckets)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.zeros(64 << 20, dtype=torch.int32, device="cuda")


def step():
    f.add_hashes(ins)
    f.find_hashes_bits(look, bits)


def timed(fn, reps=30):
    ts = []
    for _ in range(reps):
        f.clear()
        flush.zero_()
        flush_rd.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.mean(ts[5:]), min(ts)


for _ in range(5):
    step()
torch.cuda.synchronize()
print("eager  us mean/min", timed(step))
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        step()
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
torch.cuda.synchronize()
print("graph  us mean/min", timed(g.replay))
ref = bits.clone()
f.clear()
g.replay()
torch.cuda.synchronize()
print("graph result == eager:", bool(torch.equal(ref, bits)))
