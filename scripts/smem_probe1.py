"""One shared-memory lookup launch at nb, n from argv (for ncu)."""
import sys

import torch

from paper_2101_01719_b200 import SplitBlockFilter, _lib

nb, n = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda:0")
f = SplitBlockFilter(nb)
f.add_hashes(torch.randint(-2**63, 2**63 - 1, (nb * 30,), dtype=torch.int64, device=dev))
h = torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device=dev)
out = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
f.set_find_variant(_lib.FIND_SMEM)
for _ in range(3):
    f.find_hashes_bits(h, out)
torch.cuda.synchronize()
