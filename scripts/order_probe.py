import os, sys, statistics
sys.path.insert(0, "/root/repo")
import torch
from paper_2101_01719_b200 import SplitBlockFilter
from paper_2101_01719_b200 import workload as W
cfg = W.CONFIGS[4]
st = W.StreamHandle(cfg.inserts)
N, L = cfg.inserts.n, cfg.lookups.n
ins = W.gen_inserts(st, 0, N); look = W.gen_lookups(st, cfg.lookups, N, 0, L)
bits = torch.empty((L + 31) // 32, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); flush_rd = torch.zeros(64 << 20, dtype=torch.int32, device="cuda")
f = SplitBlockFilter(cfg.num_buckets); chunk = cfg.insert_chunk
def step(mid):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    f.clear(); flush.zero_(); flush_rd.sum()
    e[0].record()
    for s in range(0, N, chunk): f.add_hashes(ins[s:s + chunk])
    if mid: e[1].record()
    f.find_hashes_bits(look, bits)
    e[2].record(); torch.cuda.synchronize()
    return e[0].elapsed_time(e[2])
for _ in range(3): step(False)
for order in ([False]*4 + [True]*4, [True]*4 + [False]*4, [False, True]*4):
    r = [(m, step(m)) for m in order]
    a = statistics.mean(t for m, t in r if not m); b = statistics.mean(t for m, t in r if m)
    print("order", "".join("M" if m else "-" for m in order), f"no-mid {a:.2f} ms  mid {b:.2f} ms")
