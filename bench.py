#!/usr/bin/env python3
"""SBBF batched insert + lookup throughput on B200 (BASELINE.json metric).

A step = one pass of the hot path over one batch: insert every key of the
config's insert stream into a fresh (zeroed, untimed) filter, then look up
every key of its lookup stream (packed lookup bitmap out). Inputs are
resident in HBM before timing; L2 is flushed (256 MiB memset + 256 MiB read, untimed)
between timed steps. `value` = (inserts + lookups) / device time per step.

N = 1 (default): BASELINE config 4 — the largest single-GPU config (1e9
inserts with Zipf duplicates in 2^26-key chunks into a 1 GiB filter, then
2e9 lookups). Configs 2 and 3 are reported under `configs`.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--extra 2,3]
    python bench.py --impl reference ...   # the reference's CPU path (oracle/_ref)

N > 1 (torchrun, one rank per GPU): config 5's sharded mode — the filter is
partitioned by contiguous block range and keys are routed to their owner
rank (paper_2101_01719_b200.sharded); per-rank keys are fixed, so scaling is
weak. Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
import zlib

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SBBF insert/lookup Gkeys/s (device-timed) vs random-32B-sector roofline"
L2_FLUSH_BYTES = 256 << 20


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def golden():
    try:
        with open(os.path.join(ROOT, "tests", "golden", "configs.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def image_crc(blocks_bytes: bytes, num_buckets: int, hasher_id: int = 0) -> int:
    """FilterImage v1 trailer CRC (persist.cpp:72-88) via zlib's IEEE CRC-32."""
    hdr = b"SBBF" + bytes([1]) + hasher_id.to_bytes(4, "little") + num_buckets.to_bytes(8, "little")
    return zlib.crc32(blocks_bytes, zlib.crc32(hdr)) & 0xFFFFFFFF


# --------------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md "clocks" line)
# --------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._pump, daemon=True)
        self.thread.start()

    def _pump(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        busy = [s for s in sm if s > 0.5 * (max(sm) if sm else 0)]
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------------
# device-timed config runs
# --------------------------------------------------------------------------------
KERNEL_KINDS = ["partition", "probe_sweep", "insert_sweep", "unpermute", "tile_insert"]


def kernel_times(step, steps: int, device):
    """Live per-kernel times of the L2-blocked path: `steps` extra steps with
    the library's event pairs around every blocked launch group
    (sbbf_bench_kernel_timing), summed per kind; None when nothing blocked ran.
    These steps are not the headline's (their events add gaps)."""
    import ctypes as C

    import torch

    from paper_2101_01719_b200 import _lib
    L = _lib.lib()
    L.sbbf_bench_kernel_timing(1)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
    try:
        for k in range(steps):
            step(evs[k])
        torch.cuda.synchronize(device)
        ms = (C.c_double * len(KERNEL_KINDS))()
        n = (C.c_uint64 * len(KERNEL_KINDS))()
        rc = L.sbbf_bench_kernel_times(ms, n, len(KERNEL_KINDS))
    finally:
        L.sbbf_bench_kernel_timing(0)
    if rc != 0 or sum(n) == 0:
        return None
    t_step = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    return {"ms_per_step": t_step, "steps": steps,
            "kinds": {k: {"ms_per_step": ms[i] / steps, "launch_groups_per_step": n[i] / steps,
                          "share_of_step": ms[i] / steps / t_step}
                      for i, k in enumerate(KERNEL_KINDS) if n[i]},
            "how": "CUDA event pairs recorded by the library around each blocked-path launch group on its "
                   "stream (sbbf_bench_kernel_timing), in separate untimed steps"}


def run_config_device(cid: int, steps: int, warmup: int, device, collect_parity=True) -> dict:
    import numpy as np
    import torch

    from paper_2101_01719_b200 import SplitBlockFilter, launch_count
    from paper_2101_01719_b200 import workload as W

    cfg = W.CONFIGS[cid]
    N, L = cfg.inserts.n, cfg.lookups.n
    st = W.StreamHandle(cfg.inserts, device.index or 0)
    ins = W.gen_inserts(st, 0, N, device=device.index or 0)
    look = W.gen_lookups(st, cfg.lookups, N, 0, L, device=device.index or 0)
    bits = torch.empty((L + 31) // 32, dtype=torch.int32, device=device)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=device)
    flush_rd = torch.zeros(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=device)
    f = SplitBlockFilter(cfg.num_buckets, device=device.index or 0)
    chunk = cfg.insert_chunk or N
    stream = torch.cuda.current_stream(device)
    torch.cuda.synchronize(device)

    def flush_l2():
        # write a buffer larger than L2 (evicts everything), then read another
        # one so the lines left behind are clean: the next timed step starts
        # cold and does not pay for writing back the flush's dirty lines
        flush.zero_()
        flush_rd.sum()

    def one_step(ev):
        # ev = [start, end] times the whole step; [start, mid, end] also
        # splits it (a mid-step event blocks the programmatic launch overlap
        # of insert -> lookup, so the headline steps carry no mid event)
        ev[0].record(stream)
        for s in range(0, N, chunk):
            f.add_hashes(ins[s:s + chunk])
        if len(ev) == 3:
            ev[1].record(stream)
        f.find_hashes_bits(look, bits)
        ev[-1].record(stream)

    for _ in range(warmup):  # the same event pattern as the timed steps
        f.clear()
        flush_l2()
        one_step([torch.cuda.Event(enable_timing=True) for _ in range(2)])
    torch.cuda.synchronize(device)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
    l0 = launch_count()
    for k in range(steps):
        f.clear()
        flush_l2()  # > L2: every timed step starts cold
        one_step(evs[k])
    torch.cuda.synchronize(device)
    launches = launch_count() - l0
    t_step = [e[0].elapsed_time(e[1]) for e in evs]
    # breakdown (insert / lookup kernel time), measured in separate steps
    evb = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for k in range(steps):
        f.clear()
        flush_l2()
        one_step(evb[k])
    torch.cuda.synchronize(device)
    t_ins = [e[0].elapsed_time(e[1]) for e in evb]
    t_find = [e[1].elapsed_time(e[2]) for e in evb]
    ktimes = kernel_times(lambda ev: (f.clear(), flush_l2(), one_step(ev)), min(steps, 3), device)
    out = {
        "config": cid, "name": cfg.name, "num_buckets": cfg.num_buckets,
        "filter_bytes": cfg.filter_bytes, "inserts": N, "lookups": L,
        "insert_chunk": chunk,
        "ms_per_step": statistics.mean(t_step), "ms_insert": statistics.mean(t_ins),
        "ms_lookup": statistics.mean(t_find), "ms_step_min": min(t_step), "ms_step_max": max(t_step),
        "ms_step_median": statistics.median(t_step),
        "step_max_over_min": max(t_step) / min(t_step),
        "ms_step_split": statistics.mean(a + b for a, b in zip(t_ins, t_find)),
        "ms_steps": [round(t, 4) for t in t_step],
        "launches_per_step": launches / steps,
        "insert_variant": f.resolved_variants(chunk)[0], "find_variant": f.resolved_variants(L)[1],
    }
    if ktimes:
        out["kernel_times"] = ktimes
    out["value"] = (N + L) / (out["ms_per_step"] * 1e-3) / 1e9
    # the reference's run_bench reports the median of its reps
    # (harness.cpp:233-242): printed beside the mean
    out["value_median_step"] = (N + L) / (statistics.median(t_step) * 1e-3) / 1e9
    out["insert_gkeys_s"] = N / (out["ms_insert"] * 1e-3) / 1e9
    out["lookup_gkeys_s"] = L / (out["ms_lookup"] * 1e-3) / 1e9
    if collect_parity:
        g = golden().get(str(cid))
        blocks = f.blocks()
        crc = image_crc(blocks.tobytes(), cfg.num_buckets)
        hb = bits.cpu().numpy().view(np.uint32)
        res = np.unpackbits(hb.view(np.uint8), bitorder="little")[:L]
        j = np.arange(L, dtype=np.uint64)
        if cfg.lookups.members_first:
            mem = j < N
        else:
            mem = ((j + 1) * cfg.lookups.p // cfg.lookups.q) > (j * cfg.lookups.p // cfg.lookups.q)
        fp = int(res[~mem].sum())
        mh = int(res[mem].sum())
        par = {"image_crc": f"{crc:#010x}", "false_positives": fp, "nonmembers": int((~mem).sum()),
               "member_hits": mh, "members": int(mem.sum())}
        if g:
            par["matches_reference"] = (crc == g["image_crc"] and fp == g["false_positives"]
                                        and mh == g["members"])
        out["parity"] = par
    del f, ins, look, bits, flush, st
    torch.cuda.empty_cache()
    return out


def run_keys_frontend(steps: int, device) -> dict:
    """The XXH64 key frontend (kHasherXxh64, hash.cpp:108-114) on config 2's
    shapes: the same splitmix64 streams used as u64 KEYS, hashed inside the
    insert / lookup kernels (sbbf_gpu_insert_keys_u64 / find_keys_u64_bits).
    Device-timed like the headline step; reported, not the headline."""
    import torch

    from paper_2101_01719_b200 import SplitBlockFilter
    from paper_2101_01719_b200 import workload as W
    cfg = W.CONFIGS[2]
    N, L = cfg.inserts.n, cfg.lookups.n
    st = W.StreamHandle(cfg.inserts, device.index or 0)
    keys = W.gen_inserts(st, 0, N, device=device.index or 0)
    probes = W.gen_lookups(st, cfg.lookups, N, 0, L, device=device.index or 0)
    bits = torch.empty((L + 31) // 32, dtype=torch.int32, device=device)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=device)
    f = SplitBlockFilter(cfg.num_buckets, hasher_id=1, device=device.index or 0)
    ts = []
    for k in range(steps + 3):
        f.clear()
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f.add_keys(keys)
        f.find_keys_bits(probes, out=bits)
        e1.record()
        torch.cuda.synchronize(device)
        if k >= 3:
            ts.append(e0.elapsed_time(e1))
    ms = statistics.mean(ts)
    return {"workload": "config 2 shapes, u64 keys hashed in-kernel (XXH64 seed 0)", "ms_per_step": ms,
            "value": (N + L) / (ms * 1e-3) / 1e9, "unit": "Gkeys/s"}


def run_widened(device) -> dict:
    """SURVEY.md §8(f) rows measured beside the reference's CPU path
    (oracle/_ref, this host): the FilterImage CRC / serialize of a 1 GiB
    filter and the fpp-sim experiment. Reported, not the headline."""
    import numpy as np
    import torch

    import oracle as O
    from paper_2101_01719_b200 import SplitBlockFilter
    from paper_2101_01719_b200.fppsim import fpp_sim

    out = {}
    nb = 1 << 25  # config 4's 1 GiB
    f = SplitBlockFilter(nb, device=device.index or 0)
    f.add_keys(torch.arange(1 << 24, dtype=torch.int64, device=device))
    f.image_crc()
    torch.cuda.synchronize(device)
    t0 = time.perf_counter()
    for _ in range(5):
        f.image_crc()                      # device CRC-32 of the 1 GiB block array
    t_crc = (time.perf_counter() - t0) / 5
    t0 = time.perf_counter()
    img = f.serialize()                    # D2H of the image + device CRC
    t_ser = time.perf_counter() - t0
    del f
    sample = np.frombuffer(img, np.uint8)[: 64 << 20]
    ref = O.Reference()
    t0 = time.perf_counter()
    ref.crc32(sample.tobytes())
    t_ref = time.perf_counter() - t0
    out["image"] = {"filter_bytes": nb * 32, "gpu_crc_gbs": nb * 32 / t_crc / 1e9,
                    "gpu_serialize_gbs": len(img) / t_ser / 1e9,
                    "reference_crc_gbs": sample.size / t_ref / 1e9,
                    "reference_sample": "crc32_ieee over the first 64 MiB of the same image, 1 thread"}
    r = fpp_sim(100_000_000, 128 << 20, 10_000_000, 20160216, huge_ok=True, device=device.index or 0)
    r.pop("filter", None)
    t0 = time.perf_counter()
    fp_ref, _ = ref.fpp_sim(1_000_000, 1 << 20, 1_000_000, 20160216)
    t_ref = time.perf_counter() - t0
    out["fpp_sim"] = {"gpu": {"ndv": r["ndv"], "filter_bytes": r["filter_bytes"], "queries": r["negative_queries"],
                              "wall_s": r["wall_time_s"], "insert_mops": r["million_ops_per_sec"],
                              "measured_fpp": r["measured_fpp"], "model_fpp": r["model_fpp"]},
                      "reference": {"ndv": 1_000_000, "filter_bytes": 1 << 20, "queries": 1_000_000,
                                    "wall_s": t_ref, "ops_per_s_m": 2e6 / t_ref / 1e6,
                                    "note": "run_fpp_sim's loop on one thread (add_hash / find_hash per key)"}}
    return out


def sector_ceiling(device, filter_bytes: int, red: bool = False, n: int = 1 << 28) -> float:
    """Random 32-B sector rate (G sectors/s) on a buffer of filter_bytes."""
    import ctypes as C

    import torch

    from paper_2101_01719_b200 import _lib
    L = _lib.lib()
    buf = torch.zeros(filter_bytes // 4, dtype=torch.int32, device=device)
    sink = torch.zeros(1024, dtype=torch.int32, device=device)
    s = C.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    nb = filter_bytes // 32

    def launch(seed):
        if red:
            rc = L.sbbf_bench_sector_red(C.c_void_p(buf.data_ptr()), nb, n, seed, s)
        else:
            rc = L.sbbf_bench_sector_read(C.c_void_p(buf.data_ptr()), nb, n, seed,
                                          C.c_void_p(sink.data_ptr()), s)
        assert rc == 0
    for i in range(2):
        launch(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for i in range(3):
        e0.record()
        launch(100 + i)
        e1.record()
        torch.cuda.synchronize(device)
        times.append(e0.elapsed_time(e1))
    del buf, sink
    return n / (min(times) * 1e-3) / 1e9


def run_e2e(cid: int, steps: int, device) -> dict:
    """Same metric through the public API with HOST buffers: every step the
    library uploads the step's hashes (pinned host memory; chunked and
    overlapped with the kernels on three streams inside
    sbbf_gpu_add_hashes_host / sbbf_gpu_find_hashes_host) and downloads the
    0/1 result bytes, the reference's find_hashes output (filter.cpp:91).
    Inserts go in the config's chunks (config 4: 2^26 keys per add_hashes
    call, as the reference's batched build)."""
    import numpy as np
    import torch

    from paper_2101_01719_b200 import SplitBlockFilter
    from paper_2101_01719_b200 import workload as W

    cfg = W.CONFIGS[cid]
    N, L = cfg.inserts.n, cfg.lookups.n
    chunk = cfg.insert_chunk or N
    st = W.StreamHandle(cfg.inserts, device.index or 0)
    pinned, note = True, "pinned host arrays (torch pin_memory)"
    try:
        ins_h = torch.empty(N, dtype=torch.int64, pin_memory=True)
        look_h = torch.empty(L, dtype=torch.int64, pin_memory=True)
        res_h = torch.empty(L, dtype=torch.uint8, pin_memory=True)
    except RuntimeError as exc:  # page-locked limits: pageable arrays, the driver stages the copies
        pinned, note = False, f"pageable host arrays (pinning failed: {exc!r:.80})"
        ins_h = torch.empty(N, dtype=torch.int64)
        look_h = torch.empty(L, dtype=torch.int64)
        res_h = torch.empty(L, dtype=torch.uint8)
    # inputs generated on the device in 2^27-key pieces, copied to the host untimed
    piece = 1 << 27
    for s0 in range(0, N, piece):
        m = min(piece, N - s0)
        ins_h[s0:s0 + m].copy_(W.gen_inserts(st, s0, m, device=device.index or 0))
    for s0 in range(0, L, piece):
        m = min(piece, L - s0)
        look_h[s0:s0 + m].copy_(W.gen_lookups(st, cfg.lookups, N, s0, m, device=device.index or 0))
    torch.cuda.synchronize(device)
    ins_np = ins_h.numpy().view(np.uint64)
    look_np = look_h.numpy().view(np.uint64)
    res_np = res_h.numpy()
    f = SplitBlockFilter(cfg.num_buckets, device=device.index or 0)
    times = []
    for k in range(steps + 2):
        f.clear()
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        for s0 in range(0, N, chunk):
            f.add_hashes(ins_np[s0:s0 + chunk])   # H2D + insert kernels (synchronous)
        f.find_hashes(look_np, res_np)           # H2D + lookup kernels + D2H of the results
        t1 = time.perf_counter()
        if k >= 2:
            times.append(t1 - t0)
    hits = int(res_np.sum(dtype=np.uint64))
    del f
    # the bound e2e runs into: pinned H2D copy bandwidth (one 256 MiB copy, best of 3)
    big = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
    dbig = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        dbig.copy_(big, non_blocking=True)
        torch.cuda.synchronize(device)
        best = min(best, time.perf_counter() - t0)
    h2d_gbs = (256 << 20) / best / 1e9
    med = statistics.median(times)
    g = golden().get(str(cid))
    out = {"value": (N + L) / med / 1e9, "unit": "Gkeys/s",
           "h2d_bytes_per_step": 8 * (N + L), "d2h_bytes_per_step": L,
           "ms_per_step": med * 1e3, "steps": len(times), "hits": hits,
           "h2d_gbs_achieved": 8 * (N + L) / med / 1e9, "h2d_gbs_peak_measured": h2d_gbs,
           "bound": "PCIe host-to-device copy of the hashes (8 B/key)", "host_memory": note,
           "api": f"SplitBlockFilter.add_hashes (chunks of {chunk} keys) / find_hashes on host arrays "
                  "(sbbf_gpu_add_hashes_host / sbbf_gpu_find_hashes_host)"}
    if g:
        out["hits_match_reference"] = hits == g["member_hits"] + g["false_positives"]
    del ins_h, look_h, res_h, big, dbig
    return out


# --------------------------------------------------------------------------------
# CPU baseline: the reference itself (oracle/_ref), run_bench's method
# --------------------------------------------------------------------------------
def cpu_sample(cid: int, world: int = 1, sample_keys: int = 1 << 27):
    """(inserts, lookups, description) of the bounded CPU sample for a config.
    Configs 1-3 run in full. Config 4 (1e9 + 2e9 keys would take minutes per
    rep on one insert thread): one 2^26-key insert chunk — the first of the
    config's batched-insert chunks — into a fresh 1 GiB filter, then the
    first 2^27 lookups, the config's 1:2 insert:lookup mix. Config 5: the
    sharded arm's whole-job per-step sample (world x sample_keys each way,
    capped at 2^28), into the 8 GiB filter."""
    from paper_2101_01719_b200 import workload as W
    cfg = W.CONFIGS[cid]
    if cid == 4:
        return (1 << 26, 1 << 27,
                "config-4 sample: insert positions [0, 2^26) (the first 2^26-key chunk) into a fresh "
                "1 GiB filter, then lookup positions [0, 2^27) of the config's lookup stream")
    if cid == 5:
        n = min(sample_keys * world, 1 << 28)
        return n, n, f"a config-5 sample ({n} inserts + {n} lookups) into the 8 GiB filter"
    return cfg.inserts.n, cfg.lookups.n, f"config {cid} in full"


def cpu_reference_run(cid: int, reps: int, threads: int, world: int = 1, sample_keys: int = 1 << 27,
                      warmup: int = 0) -> dict:
    """The reference core itself (oracle/_ref, run_bench's method,
    harness.cpp:132-245) on the bounded sample of `cpu_sample`. The first
    `warmup` reps run untimed (dropped)."""
    import dataclasses

    import numpy as np

    import oracle as O
    from paper_2101_01719_b200 import workload as W

    cfg = W.CONFIGS[cid]
    N, L, what = cpu_sample(cid, world, sample_keys)
    ins_spec = cfg.inserts
    num_inserts = cfg.inserts.n
    if cid == 5:
        ins_spec = dataclasses.replace(cfg.inserts, n=N)
        num_inserts = N
    orc = O.Oracle()
    table = W.zipf_cdf_table(cfg.inserts.zipf_s, cfg.inserts.zipf_n) if cfg.inserts.dup_num else None
    ost = orc.stream(ins_spec, table)
    ins = orc.gen_inserts(ost, 0, N)
    look = orc.gen_lookups(ost, cfg.lookups, num_inserts, 0, L)
    try:
        ref = O.Reference()
        kind = "reference"
        ti, tl, res, blocks = ref.time_build_probe(cfg.num_buckets, ins, look, threads, warmup + reps)
        ti, tl = ti[warmup:], tl[warmup:]
        # lookups on one core as well as on all of them
        tl1 = ref.time_build_probe(cfg.num_buckets, ins, look, 1, 1)[1] if threads > 1 and cid < 5 else tl
    except (FileNotFoundError, OSError):
        kind = "port"
        ti, tl = [], []
        for r in range(warmup + reps):
            b = orc.new_blocks(cfg.num_buckets)
            t0 = time.perf_counter()
            orc.add_hashes(b, ins)
            ti.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            res = orc.find_hashes(b, look, threads)
            tl.append(time.perf_counter() - t0)
            if r < warmup:
                ti.pop()
                tl.pop()
        blocks = b
        tl1 = tl
    mi, ml = statistics.median(ti), statistics.median(tl)
    # image CRC only for the configs run in full (their goldens exist)
    full = cid in (1, 2, 3)
    crc = image_crc(np.ascontiguousarray(blocks).tobytes(), cfg.num_buckets) if full else None
    return {"value": (N + L) / (mi + ml) / 1e9, "unit": "Gkeys/s", "cores": threads, "kind": kind,
            "sample": f"{what}, median of {reps} reps; "
                      f"insert 1 thread (the reference's only writer mode), lookup {threads} "
                      f"jthreads (harness.cpp:173-200); -O3 -DNDEBUG, AVX2 backend",
            "inserts": N, "lookups": L,
            "insert_gkeys_s": N / mi / 1e9, "lookup_gkeys_s": L / ml / 1e9,
            "lookup_gkeys_s_1thread": L / statistics.median(tl1) / 1e9,
            "image_crc": f"{crc:#010x}" if crc is not None else None, "hits": int(res.sum(dtype=np.uint64))}


def run_reference_arm(args) -> None:
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    world = env_int("WORLD_SIZE", 1)
    reps = max(args.steps, 1)
    r = cpu_reference_run(args.config, reps, threads, world=world, sample_keys=args.sample_keys,
                          warmup=args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": "Gkeys/s",
        "n_gpus": args.gpus, "steps": reps, "warmup": args.warmup,
        "ms_per_step": (r["inserts"] + r["lookups"]) / r["value"] / 1e6,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded splitmix64 hash streams, BASELINE.json)",
        "config": workload_config(args.config, world, args.sample_keys),
        "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": r["value"], "unit": "Gkeys/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "insert_gkeys_s": r["insert_gkeys_s"], "lookup_gkeys_s": r["lookup_gkeys_s"],
        "lookup_gkeys_s_1thread": r["lookup_gkeys_s_1thread"],
        "image_crc": r["image_crc"],
    }
    print(json.dumps(line), flush=True)


def workload_config(cid: int, world: int = 1, sample_keys: int = 1 << 27) -> dict:
    """The `config` object of both arms (identical for the same command)."""
    from paper_2101_01719_b200 import workload as W
    cfg = W.CONFIGS[cid]
    if cid == 5:
        return {"workload": f"BASELINE config 5 sample: 8 GiB filter ({cfg.num_buckets} blocks) sharded over "
                            f"{world} rank(s) by block range; per rank per step {sample_keys:,} inserts "
                            f"+ {sample_keys:,} lookups (25% members)", "config_id": cid,
                "inserts_per_rank": sample_keys, "lookups_per_rank": sample_keys,
                "num_buckets": cfg.num_buckets, "parallelism": f"shard{world}",
                "l2": "flushed between timed steps (untimed)"}
    c = {"workload": f"BASELINE config {cid}: {cfg.inserts.n:,} inserts into "
                     f"{cfg.filter_bytes:,} B ({cfg.num_buckets} blocks), then "
                     f"{cfg.lookups.n:,} lookups", "config_id": cid,
         "inserts": cfg.inserts.n, "lookups": cfg.lookups.n, "num_buckets": cfg.num_buckets,
         "l2": "flushed between timed steps (256 MiB memset then 256 MiB read, untimed)",
         "lookup_output": "packed bitmap (1 bit/key)", "parallelism": "single GPU"}
    if cfg.insert_chunk:
        c["insert_chunk"] = cfg.insert_chunk
    return c


def ncu_traffic(cid: int, phase: str, keys: int):
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of one
    phase (`lookup` / `insert`: every kernel the phase launches) from the
    committed ncu launch lists (profiles/traffic.json), per key, scaled to
    this run's keys; None when no capture exists."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)[str(cid)][phase]
    except Exception:
        return None, None
    return t["dram_bytes_per_key"] * keys, t


def lookup_split(filter_bytes: int, l2_bytes: int) -> bool:
    """sbbf_kernels.cu split_log2 for lookups: whole filters in (0.6, 1.2] x L2
    are probed in two range-split passes."""
    return 0.6 * l2_bytes < filter_bytes <= 1.2 * l2_bytes


def roofline(res: dict, hbm_peak: float, peak_note: str, l2_bytes: int, l2_read_gs: float,
             l2_red_gs: float) -> tuple[dict, dict]:
    """The north star's roofline: one random 32-byte sector per key (read
    for a lookup, read-modify-write = 64 B for an insert) at HBM bandwidth —
    or, for a filter that fits in L2, at the L2 random-sector rate measured
    on a filter-sized buffer (sbbf_bench_sector_read / _red: MEASURED_PEAKS
    has no L2 figure). achieved = keys x 32 (64) B / phase time; frac =
    achieved / peak. The streamed bytes the kernels actually move (hashes,
    partition passes, bitmap) are reported under `stream` and, measured by
    ncu, as `traffic`."""
    L, N = res["lookups"], res["inserts"]
    t_l, t_i = res["ms_lookup"] * 1e-3, res["ms_insert"] * 1e-3
    resident = res["filter_bytes"] <= l2_bytes // 2
    if resident:
        peak_l = l2_read_gs * 32.0
        peak_i = l2_red_gs * 64.0
        pnote = ("L2: random 32-B sector rate measured in this run on a filter-sized buffer "
                 f"({l2_read_gs:.1f} G sectors/s read, {l2_red_gs:.1f} G/s red; sbbf_bench_sector_*), "
                 "x 32 B (lookup) / x 64 B (insert)")
        bound = "l2"
    else:
        peak_l = peak_i = hbm_peak
        pnote = peak_note
        bound = "hbm"
    kernels = {1: "find_whole_kernel / find_split_kernel (direct, bitmap)", 2: "find_smem_kernel",
               3: "blocked: partition + slice sweep (sbbf_blocked.cu)"}
    ach_l = L * 32.0 / t_l / 1e9
    traffic, tl = ncu_traffic(res["config"], "lookup", L)
    rl = {"bound": bound, "kernel": kernels.get(res.get("find_variant"), "lookup"),
          "achieved": ach_l, "peak": peak_l, "unit": "GB/s", "frac": ach_l / peak_l,
          "traffic": traffic, "bytes_per_key": 32.0,
          "ceiling_gkeys_s": peak_l / 32.0, "lookup_gkeys_s": L / t_l / 1e9,
          "peak_note": pnote,
          "bytes_note": "north-star roofline: one random 32-B sector read per lookup",
          "traffic_note": ("ncu dram__bytes_read.sum + dram__bytes_write.sum of every kernel of the lookup "
                           f"phase ({tl['source']}), {tl['dram_bytes_per_key']:.2f} B/key x {L} lookups"
                           if tl else "no ncu capture committed for this config")}
    ach_i = N * 64.0 / t_i / 1e9
    traffic_i, ti = ncu_traffic(res["config"], "insert", N)
    ri = {"bound": bound, "achieved": ach_i, "peak": peak_i, "unit": "GB/s", "frac": ach_i / peak_i,
          "traffic": traffic_i, "bytes_per_key": 64.0, "ceiling_gkeys_s": peak_i / 64.0,
          "insert_gkeys_s": N / t_i / 1e9, "peak_note": pnote,
          "bytes_note": "north-star roofline: read-modify-write of one random 32-B sector per insert",
          "traffic_note": ("ncu DRAM bytes of every kernel of the insert phase "
                           f"({ti['source']}), {ti['dram_bytes_per_key']:.2f} B/key" if ti else
                           "no ncu capture committed for this config")}
    kt = res.get("kernel_times")
    if kt:
        rl["dominant_kernel"], rl["kernels"] = kernel_rooflines(res, kt, hbm_peak)
    return rl, ri


# SM count and clock of the part: the L2->SM sector port moves one 32-B sector
# per SM-clock (148 x 1.965 GHz = 290.8 G sectors/s; the round-1 microbenchmark
# measured 288 G/s for random 32-B reads of an L2-resident buffer).
SMS, SM_GHZ = 148, 1.965


def kernel_rooflines(res: dict, kt: dict, hbm_peak: float):
    """Each blocked-path kernel kind against its own bound, from the live
    per-kind times (kernel_times): achieved = algorithmic bytes (or sectors)
    per launch group / its average live duration. The dominant kind is the
    one with the largest share of the step."""
    N, L = res["inserts"], res["lookups"]
    port_peak = SMS * SM_GHZ  # G sectors/s
    out = {}
    for kind, v in kt["kinds"].items():
        groups, ms = v["launch_groups_per_step"], v["ms_per_step"]
        avg_ms = ms / groups
        d = {"launch_groups_per_step": groups, "avg_launch_group_ms": avg_ms, "share_of_step": v["share_of_step"]}
        if kind == "probe_sweep":
            keys = L / groups
            d.update({"keys_per_launch": keys, "bound": "L2->SM sector port (1 sector / SM-clock)",
                      "algorithmic": "one 32-B probe sector + 8-B key per lookup (1.25 sectors)",
                      "achieved_gsectors_s": keys * 1.25 / (avg_ms * 1e-3) / 1e9, "peak_gsectors_s": port_peak,
                      "frac": keys * 1.25 / (avg_ms * 1e-3) / 1e9 / port_peak,
                      "north_star_gbs": keys * 32 / (avg_ms * 1e-3) / 1e9})
        elif kind == "insert_sweep":
            keys = N / groups
            d.update({"keys_per_launch": keys, "bound": "L2 test-and-red rate (DESIGN.md section 3)",
                      "achieved_gkeys_s": keys / (avg_ms * 1e-3) / 1e9,
                      "north_star_gbs": keys * 64 / (avg_ms * 1e-3) / 1e9,
                      "north_star_frac": keys * 64 / (avg_ms * 1e-3) / 1e9 / hbm_peak})
        elif kind == "partition":
            # every insert call and lookup round: keys read once, written bucket-major;
            # the unfused lookups (an unpermute kind in the times) also write 2-B positions
            byts = (N * 16 + L * (18 if "unpermute" in kt["kinds"] else 16)) / groups
            d.update({"bound": "hbm", "algorithmic_bytes_per_launch": byts,
                      "achieved_gbs": byts / (avg_ms * 1e-3) / 1e9, "peak_gbs": hbm_peak,
                      "frac": byts / (avg_ms * 1e-3) / 1e9 / hbm_peak})
        elif kind == "unpermute":
            byts = L * (1 + 2 + 1 / 8) / groups
            d.update({"bound": "hbm", "algorithmic_bytes_per_launch": byts,
                      "achieved_gbs": byts / (avg_ms * 1e-3) / 1e9, "peak_gbs": hbm_peak,
                      "frac": byts / (avg_ms * 1e-3) / 1e9 / hbm_peak})
        out[kind] = d
    dom = max(out, key=lambda k: out[k]["share_of_step"])
    return dict(kernel=dom, **out[dom]), out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=None,
                    help="4 (default, single GPU) / 2 / 3; under torchrun the default is 5 (sharded)")
    ap.add_argument("--sample-keys", type=int, default=1 << 27,
                    help="config 5: inserts and lookups per rank per step (bounded sample)")
    ap.add_argument("--extra", default="2,3", help="extra configs reported under 'configs'")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-widened", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="run the multi-GPU sharded path even at world size 1")
    ap.add_argument("--route", default="auto", choices=["auto", "fused", "nccl"],
                    help="sharded key routing: fused peer-memory dispatch or NCCL all-to-all")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.config is None:
        args.config = 5 if env_int("WORLD_SIZE", 1) > 1 else 4
    if args.impl == "reference":
        run_reference_arm(args)
        return

    world = env_int("WORLD_SIZE", 1)
    if world > 1 or args.sharded or args.config == 5:
        from paper_2101_01719_b200 import sharded
        rank = env_int("RANK", 0)
        clocks = ClockSampler(env_int("LOCAL_RANK", 0))
        if rank == 0:
            clocks.start()
        line = sharded.bench_main(args)
        if rank == 0:
            line["clocks"] = clocks.stop()
            if args.config == 5:
                line["config"] = dict(workload_config(5, world, args.sample_keys),
                                      routing=line["config"].get("workload", ""))
                if not args.no_cpu_baseline and world == 1:
                    try:
                        cb = cpu_reference_run(5, 1, os.cpu_count() or 1, world=1, sample_keys=args.sample_keys)
                        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                                   "insert_gkeys_s", "lookup_gkeys_s")}
                    except Exception as exc:  # the baseline never blocks the GPU line
                        line["cpu_baseline"] = {"value": None, "error": repr(exc)}
            print(json.dumps(line), flush=True)
        return

    import torch
    device = torch.device("cuda", env_int("LOCAL_RANK", 0))
    torch.cuda.set_device(device)
    hbm_peak, peak_note = measured_peaks()
    props = torch.cuda.get_device_properties(device)
    l2_bytes = getattr(props, "L2_cache_size", 126 << 20)

    clocks = ClockSampler(device.index or 0)
    clocks.start()
    main_res = run_config_device(args.config, args.steps, args.warmup, device)
    clk = clocks.stop()
    extras = {}
    for c in [int(x) for x in args.extra.split(",") if x.strip()]:
        if c == args.config or c not in (1, 2, 3, 4):
            continue
        extras[str(c)] = run_config_device(c, max(3, min(args.steps, 5)), 3, device)

    # L2 random-sector ceilings (the roofline denominators of L2-resident filters)
    ceil = {}
    for r in [main_res] + list(extras.values()):
        fb = max(r["filter_bytes"], 1 << 20)
        if fb <= l2_bytes // 2 and fb not in ceil:
            ceil[fb] = (sector_ceiling(device, fb), sector_ceiling(device, fb, red=True))
    for r in [main_res] + list(extras.values()):
        l2r, l2w = ceil.get(max(r["filter_bytes"], 1 << 20), (None, None))
        r["roofline"], r["insert_roofline"] = roofline(r, hbm_peak, peak_note, l2_bytes, l2r or 0.0, l2w or 0.0)

    line = {
        "metric": METRIC, "value": main_res["value"], "unit": "Gkeys/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": main_res["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded splitmix64 hash streams of BASELINE.json, generated in HBM)",
        "config": workload_config(args.config),
        "value_median_step": main_res["value_median_step"],
        "ms_step_median": main_res["ms_step_median"], "ms_step_min": main_res["ms_step_min"],
        "ms_step_max": main_res["ms_step_max"], "step_max_over_min": main_res["step_max_over_min"],
        "insert_gkeys_s": main_res["insert_gkeys_s"], "lookup_gkeys_s": main_res["lookup_gkeys_s"],
        "ms_insert": main_res["ms_insert"], "ms_lookup": main_res["ms_lookup"],
        "step_timing": ("value/ms_per_step: mean of the K timed steps, CUDA events at step start and end "
                        "only; ms_insert/ms_lookup: separate steps with a mid-step event "
                        f"(their sum {main_res['ms_step_split']:.4f} ms)"),
        "roofline": main_res["roofline"], "insert_roofline": main_res["insert_roofline"],
        "gpu_launches": int(round(main_res["launches_per_step"] * args.steps)),
        "launches_per_step": main_res["launches_per_step"],
        "clocks": clk, "parity": main_res.get("parity"),
        "variants": {"insert": main_res["insert_variant"], "find": main_res["find_variant"]},
        "configs": {k: {kk: v for kk, v in r.items() if kk not in ("name",)}
                    for k, r in extras.items()},
    }
    if not args.no_widened:
        try:
            line["keys_frontend"] = run_keys_frontend(max(3, min(args.steps, 10)), device)
            line["widened"] = run_widened(device)
        except Exception as exc:  # the extra rows never block the headline line
            line["widened"] = {"error": repr(exc)}
    if not args.no_e2e:
        try:
            line["e2e"] = run_e2e(args.config, 3, device)
        except Exception as exc:  # reported, never blocks the line
            line["e2e"] = {"value": None, "error": repr(exc)}
    if not args.no_cpu_baseline:
        try:
            cb = cpu_reference_run(args.config, 3, os.cpu_count() or 1)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "insert_gkeys_s",
                                                       "lookup_gkeys_s", "lookup_gkeys_s_1thread")}
            line["cpu_baseline"]["image_crc"] = cb["image_crc"]
        except Exception as exc:  # the baseline never blocks the GPU line
            line["cpu_baseline"] = {"value": None, "error": repr(exc)}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
