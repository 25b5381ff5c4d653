"""GPU false-positive experiment — the reference's ``sbbf fpp-sim``
(``tools/harness.cpp:67-109``, run_fpp_sim) on device.

Keys are the counters ``[0, ndv)`` hashed with ``hash_u64_key(c, seed)``
(KeyMode::kRandom64, ``harness.cpp:60-65``; XXH64 fused into the insert
kernel); probes are the disjoint counters ``[2^32, 2^32 + q)``, so every hit
is a false positive. The filter records ``kHasherXxh64`` (= 1) as its hasher
id, as the reference does (``harness.cpp:85``). The false-positive COUNT is
bit-identical to the reference's for the same arguments (tests).
"""
from __future__ import annotations

import time

from .filter import SplitBlockFilter
from .tools import sbbf_fpp  # noqa: F401  (model.cpp:78-103, bit-exact restatement)

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None

NEGATIVE_COUNTER_BASE = 1 << 32      # harness.cpp:31
HUGE_NDV_THRESHOLD = 10_000_000      # harness.hpp:85
KHASHER_XXH64 = 1                    # hash.hpp:12


def fpp_sim(ndv: int, filter_bytes: int, negative_queries: int = 1_000_000, seed: int = 1,
            huge_ok: bool = False, device: int = 0, chunk: int = 1 << 26) -> dict:
    """run_fpp_sim on the GPU. Raises ValueError where the reference throws
    UsageError (harness.cpp:36-56, 73-78)."""
    if filter_bytes < 32:
        raise ValueError("--bytes must be at least 32 (one block)")
    if ndv > NEGATIVE_COUNTER_BASE:
        raise ValueError("--ndv must not exceed 2^32 (the negative-query key space starts there)")
    if ndv > HUGE_NDV_THRESHOLD and not huge_ok:
        raise ValueError("--ndv beyond 10M is paper scale; pass --huge to allow it")
    if negative_queries < 1:
        raise ValueError("--queries must be positive")
    if negative_queries > NEGATIVE_COUNTER_BASE:
        raise ValueError("--queries must not exceed 2^32")
    buckets = filter_bytes // 32
    dev = torch.device("cuda", device)
    f = SplitBlockFilter(buckets, hasher_id=KHASHER_XXH64, device=device)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for s in range(0, ndv, chunk):
        f.add_keys(torch.arange(s, min(s + chunk, ndv), dtype=torch.int64, device=dev), seed)
    e1.record()
    fp = 0
    for s in range(0, negative_queries, chunk):
        q = torch.arange(NEGATIVE_COUNTER_BASE + s, NEGATIVE_COUNTER_BASE + min(s + chunk, negative_queries),
                         dtype=torch.int64, device=dev)
        fp += int(f.find_keys(q, seed).sum(dtype=torch.int64).item())
    wall = time.perf_counter() - t0
    insert_ms = e0.elapsed_time(e1)
    return {
        "op": "fpp-sim", "ndv": ndv, "filter_bytes": buckets * 32, "false_positives": fp,
        "negative_queries": negative_queries,
        "measured_fpp": fp / negative_queries,
        "model_fpp": sbbf_fpp(ndv / buckets),
        "million_ops_per_sec": ndv / (insert_ms * 1e-3) / 1e6 if insert_ms > 0 else 0.0,
        "wall_time_s": wall,
        "filter": f,
    }
