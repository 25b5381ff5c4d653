"""Times the device CRC-32 of a 1 GiB block array (image_crc) for ncu runs."""
import time

import torch

from paper_2101_01719_b200 import SplitBlockFilter

f = SplitBlockFilter(1 << 25)
f.add_hashes(torch.randint(-2**63, 2**63 - 1, (1 << 24,), dtype=torch.int64, device="cuda"))
for _ in range(3):
    f.image_crc()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    f.image_crc()
print("image_crc GB/s", (1 << 30) * 10 / (time.perf_counter() - t0) / 1e9)
