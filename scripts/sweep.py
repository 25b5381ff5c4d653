#!/usr/bin/env python3
"""Kernel-variant and random-sector sweeps on one GPU (design evidence).

    python scripts/sweep.py sectors   # random 32-B sector read/red rate vs buffer size
    python scripts/sweep.py variants  # insert/find variants per BASELINE config

Prints a table and writes JSON to gpurun_out/sweep_<mode>.json. Device-timed
with CUDA events; L2 flushed (256 MiB memset) before every timed launch.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2101_01719_b200 import SplitBlockFilter, _lib  # noqa: E402
from paper_2101_01719_b200 import workload as W  # noqa: E402

DEV = torch.device("cuda:0")
FLUSH = None


def flush():
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device=DEV)
    FLUSH.zero_()


def timed(fn, reps=5, warm=2, do_flush=True):
    for _ in range(warm):
        if do_flush:
            flush()
        fn()
    ts = []
    for _ in range(reps):
        if do_flush:
            flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def sectors():
    L = _lib.lib()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    sink = torch.zeros(1024, dtype=torch.int32, device=DEV)
    out = []
    n = 1 << 28
    for gran in (None, 32, 64, 128):
        old = C.c_int(0)
        if gran is not None:
            _lib.check(L.sbbf_gpu_set_l2_fetch_granularity(0, gran, C.byref(old)), "gran")
        for mb in (1, 16, 64, 128, 256, 512, 1024, 4096, 16384):
            buf = torch.zeros((mb << 20) // 4, dtype=torch.int32, device=DEV)
            nb = (mb << 20) // 32
            t_rd = timed(lambda: L.sbbf_bench_sector_read(C.c_void_p(buf.data_ptr()), nb, n, 7,
                                                          C.c_void_p(sink.data_ptr()), s))
            t_red = timed(lambda: L.sbbf_bench_sector_red(C.c_void_p(buf.data_ptr()), nb, n, 9, s))
            r = {"gran": gran, "buf_mib": mb, "read_gs": n / t_rd / 1e6, "red_gs": n / t_red / 1e6}
            out.append(r)
            print(f"gran={gran} buf={mb:6d} MiB  read {r['read_gs']:7.1f} G/s  red {r['red_gs']:7.1f} G/s",
                  flush=True)
            del buf
        if gran is not None:
            L.sbbf_gpu_set_l2_fetch_granularity(0, old.value, None)
    return out


def variants():
    out = []
    for cid in (1, 2, 3, 4):
        cfg = W.CONFIGS[cid]
        st = W.StreamHandle(cfg.inserts)
        N, Lk = cfg.inserts.n, cfg.lookups.n
        ins = W.gen_inserts(st, 0, N)
        look = W.gen_lookups(st, cfg.lookups, N, 0, Lk)
        bits = torch.empty((Lk + 31) // 32, dtype=torch.int32, device=DEV)
        byts = torch.empty(Lk, dtype=torch.uint8, device=DEV)
        f = SplitBlockFilter(cfg.num_buckets)
        chunk = cfg.insert_chunk or N
        for iv, name in ((1, "lane8"), (2, "lane8_test"), (3, "thread"), (4, "wide"), (5, "wide_test"),
                         (6, "blocked")):
            f.set_insert_variant(iv)

            def ins_fn():
                f.clear()
                for s0 in range(0, N, chunk):
                    f.add_hashes(ins[s0:s0 + chunk])
            # clear is a memset (tiny vs the inserts); included in both arms alike
            t = timed(ins_fn, reps=3 if cid >= 3 else 7)
            r = {"config": cid, "op": "insert", "variant": name, "ms": t, "gkeys_s": N / t / 1e6}
            out.append(r)
            print(f"cfg{cid} insert {name:11s} {t:9.3f} ms {r['gkeys_s']:8.2f} Gkeys/s", flush=True)
        f.set_insert_variant(0)
        f.clear()
        for s0 in range(0, N, chunk):
            f.add_hashes(ins[s0:s0 + chunk])
        fvs = [(1, "global"), (3, "blocked")] + ([(2, "smem")] if cfg.filter_bytes <= 200 * 1024 else [])
        for fv, name in fvs:
            f.set_find_variant(fv)
            for kind, fn in (("bits", lambda: f.find_hashes_bits(look, bits)),
                             ("bytes", lambda: f.find_hashes(look, byts))):
                t = timed(fn, reps=3 if cid >= 3 else 7)
                r = {"config": cid, "op": f"find_{kind}", "variant": name, "ms": t, "gkeys_s": Lk / t / 1e6}
                out.append(r)
                print(f"cfg{cid} find-{kind:5s} {name:11s} {t:9.3f} ms {r['gkeys_s']:8.2f} Gkeys/s", flush=True)
        del f, ins, look, bits, byts, st
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "variants"
    res = {"sectors": sectors, "variants": variants}[mode]()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"sweep_{mode}.json"), "w") as fh:
        json.dump(res, fh, indent=1)
