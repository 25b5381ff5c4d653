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


def resolve_buckets(ndv: int, filter_bytes: int | None, target_fpp: float | None) -> int:
    """harness.cpp:33-47: exactly one of --bytes / --fpp."""
    from .tools import size_for
    if (filter_bytes is None) == (target_fpp is None):
        raise ValueError("exactly one of --bytes or --fpp must be given")
    if filter_bytes is not None:
        if filter_bytes < 32:
            raise ValueError("--bytes must be at least 32 (one block)")
        return filter_bytes // 32
    if not (0.0 < target_fpp < 1.0):
        raise ValueError("--fpp must lie strictly between 0 and 1")
    return 1 if ndv == 0 else size_for(ndv, target_fpp)


def fpp_sim(ndv: int, filter_bytes: int | None = None, negative_queries: int = 1_000_000, seed: int = 1,
            huge_ok: bool = False, device: int = 0, chunk: int = 1 << 26, target_fpp: float | None = None,
            key_mode: str = "random64") -> dict:
    """run_fpp_sim on the GPU. Raises ValueError where the reference throws
    UsageError (harness.cpp:33-56, 73-78). key_mode "random64" hashes the
    counters as u64 keys (fused into the kernels), "strings" hashes their
    decimal strings (hash_key(std::to_string(c)), on the device)."""
    if key_mode not in ("random64", "strings"):
        raise ValueError("--key-mode must be 'random64' or 'strings'")
    if ndv > NEGATIVE_COUNTER_BASE:
        raise ValueError("--ndv must not exceed 2^32 (the negative-query key space starts there)")
    if ndv > HUGE_NDV_THRESHOLD and not huge_ok:
        raise ValueError("--ndv beyond 10M is paper scale; pass --huge to allow it")
    if negative_queries < 1:
        raise ValueError("--queries must be positive")
    if negative_queries > NEGATIVE_COUNTER_BASE:
        raise ValueError("--queries must not exceed 2^32")
    buckets = resolve_buckets(ndv, filter_bytes, target_fpp)
    try:
        model = sbbf_fpp(ndv / buckets)
    except ValueError:
        raise ValueError("--bytes is far too small for --ndv; the model only covers a <= 1e6") from None
    dev = torch.device("cuda", device)
    f = SplitBlockFilter(buckets, hasher_id=KHASHER_XXH64, device=device)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    from .filter import hash_counter_strings
    for s in range(0, ndv, chunk):
        m = min(s + chunk, ndv) - s
        if key_mode == "random64":
            f.add_keys(torch.arange(s, s + m, dtype=torch.int64, device=dev), seed)
        else:
            f.add_hashes(hash_counter_strings(s, m, seed, device))
    e1.record()
    fp = 0
    for s in range(0, negative_queries, chunk):
        m = min(s + chunk, negative_queries) - s
        if key_mode == "random64":
            q = torch.arange(NEGATIVE_COUNTER_BASE + s, NEGATIVE_COUNTER_BASE + s + m, dtype=torch.int64, device=dev)
            fp += int(f.find_keys(q, seed).sum(dtype=torch.int64).item())
        else:
            fp += int(f.find_hashes(hash_counter_strings(NEGATIVE_COUNTER_BASE + s, m, seed, device))
                      .sum(dtype=torch.int64).item())
    wall = time.perf_counter() - t0
    insert_ms = e0.elapsed_time(e1)
    return {
        "op": "fpp-sim", "ndv": ndv, "filter_bytes": buckets * 32, "false_positives": fp,
        "negative_queries": negative_queries,
        "measured_fpp": fp / negative_queries,
        "model_fpp": model,
        "million_ops_per_sec": ndv / (insert_ms * 1e-3) / 1e6 if insert_ms > 0 else 0.0,
        "wall_time_s": wall,
        "filter": f,
    }


def sbbf_fpp_mc(a: float, blocks: int, trials: int, seed: int = 0, device: int = 0) -> float:
    """The reference's Monte-Carlo oracle (model.cpp:105-128) on the GPU:
    Poisson(a) keys per block drawn from the block's preimage interval, then
    `trials` uniform probes. Counter-based per-block streams (not the
    reference's mt19937_64 draws): the same experiment, seed-reproducible.
    Raises ValueError where the reference throws std::domain_error."""
    import ctypes as C

    from . import _lib
    out = C.c_double(0.0)
    rc = _lib.lib().sbbf_gpu_fpp_mc(float(a), int(blocks), int(trials), int(seed), int(device), C.byref(out))
    if rc == _lib.SBBF_EINVAL:
        raise ValueError(_lib.lib().sbbf_gpu_last_error().decode())
    _lib.check(rc, "sbbf_gpu_fpp_mc")
    return out.value
