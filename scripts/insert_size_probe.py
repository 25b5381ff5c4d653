#!/usr/bin/env python3
"""Blocked insert sweep rate against filter size: 15 calls of 2^26 distinct
keys into filters of 64 MiB .. 4 GiB (forced BLOCKED), device-timed, with the
per-kernel split from the library's event timing.

    python scripts/insert_size_probe.py
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2101_01719_b200 import SplitBlockFilter, _lib  # noqa: E402
from paper_2101_01719_b200 import workload as W  # noqa: E402

CH = 1 << 26
ins = W.gen_inserts(W.StreamHandle(W.InsertSpec(seed=7, n=15 * CH)), 0, 15 * CH)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
L = _lib.lib()
for lg in (21, 22, 23, 24, 25, 26, 27):
    nb = 1 << lg
    f = SplitBlockFilter(nb)
    f.set_insert_variant(_lib.INSERT_BLOCKED)
    for rep in range(3):
        f.clear()
        flush.zero_()
        if rep == 2:
            L.sbbf_bench_kernel_timing(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in range(0, 15 * CH, CH):
            f.add_hashes(ins[s:s + CH])
        e1.record()
        torch.cuda.synchronize()
    ms = (C.c_double * 5)()
    n = (C.c_uint64 * 5)()
    L.sbbf_bench_kernel_times(ms, n, 5)
    L.sbbf_bench_kernel_timing(0)
    t = e0.elapsed_time(e1)
    sweep = ms[2] / max(n[2], 1)
    print(f"filter {nb * 32 >> 20:6d} MiB  phase {15 * CH / t / 1e6:6.1f} Gkeys/s  sweep/call {sweep:.3f} ms "
          f"({CH / sweep / 1e6:6.1f} Gkeys/s)  partition/call {ms[0] / max(n[0], 1):.3f} ms", flush=True)
    del f
