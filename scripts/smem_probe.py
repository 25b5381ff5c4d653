"""Lookup rate of the shared-memory lookup (filter cut into parts that fit
one CTA's shared memory) vs the global pipelined lookup, and their agreement."""
import torch

from paper_2101_01719_b200 import SplitBlockFilter, _lib

dev = torch.device("cuda:0")
for nb in (4096, 32768, 65536, 8 * 7000):
    f = SplitBlockFilter(nb)
    f.add_hashes(torch.randint(-2**63, 2**63 - 1, (nb * 30,), dtype=torch.int64, device=dev))
    for n in (10_000_000, 100_000_000):
        h = torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device=dev)
        res = {}
        for name, v in (("global", _lib.FIND_GLOBAL), ("smem", _lib.FIND_SMEM)):
            try:
                f.set_find_variant(v)
            except Exception as exc:
                print(nb, name, exc)
                continue
            out = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
            for _ in range(3):
                f.find_hashes_bits(h, out)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            for _ in range(10):
                f.find_hashes_bits(h, out)
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / 10
            res[name] = out.clone()
            byt = f.find_hashes(h[:1_000_003])
            print(f"nb={nb} n={n} {name}: {ms:.4f} ms  {n / ms / 1e6:.1f} Gkeys/s  bytes_sum={int(byt.sum())}")
        if len(res) == 2:
            print("  agree:", bool(torch.equal(res["global"], res["smem"])))
