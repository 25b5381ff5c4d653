#!/usr/bin/env python3
"""Random 32-byte sector read rate against the size of the window read
(sbbf_bench_sector_read: 8 loads in flight per thread, 4 CTAs x 256 threads per
SM, no hash stream): the rate the blocked lookup sweep could reach on an
L2-resident slice of each size, and how it falls as the window leaves L2.

    python scripts/l2_window_probe.py [MiB ...]
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2101_01719_b200 import _lib  # noqa: E402

L = _lib.lib()
sizes = [int(x) for x in sys.argv[1:]] or [1, 4, 8, 16, 32, 48, 64, 96, 128, 256, 1024]
sink = torch.zeros(1024, dtype=torch.int32, device="cuda")
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
n = 1 << 28
for mb in sizes:
    nb = (mb << 20) // 32
    buf = torch.zeros(nb * 8, dtype=torch.int32, device="cuda")
    for i in range(2):  # warm: the window is in L2 (if it fits) before the timed launches
        assert L.sbbf_bench_sector_read(C.c_void_p(buf.data_ptr()), nb, n, 7 + i, C.c_void_p(sink.data_ptr()), s) == 0
    ts = []
    for i in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert L.sbbf_bench_sector_read(C.c_void_p(buf.data_ptr()), nb, n, 100 + i, C.c_void_p(sink.data_ptr()), s) == 0
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[1]
    print(f"window {mb:5d} MiB: {n / t / 1e6:7.1f} G sectors/s ({n * 32 / t / 1e6:7.0f} GB/s), median of 3 x 2^28 random reads, {t:.3f} ms")
    del buf
