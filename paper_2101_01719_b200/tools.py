"""Batch build / query from key files on the GPU — the reference's
``sbbf build`` and ``sbbf query`` (tools/harness.cpp:247-304), plus the
sizing model they use (core/src/model.cpp:78-103,170-212).

    python -m paper_2101_01719_b200.tools build KEYS OUT.sbbf --fpp 0.01
    python -m paper_2101_01719_b200.tools query OUT.sbbf KEYS      # maybe/absent per line

Keys are the newline-separated segments of the file (a final segment without
a newline is a key; read_key_lines, harness.cpp:247-260), hashed with XXH64
seed 0 (hash_key, hasher id 1) on the GPU; the image is the v1 FilterImage,
so a filter built here loads in the reference and vice versa.
"""
from __future__ import annotations

import argparse
import math
import sys

import numpy as np

from .filter import SplitBlockFilter, hash_keys

KHASHER_XXH64 = 1

# The C library's lgamma (what std::lgamma calls); CPython's math.lgamma is
# its own implementation and differs from glibc in the last ulp.
try:
    import ctypes as _C
    import ctypes.util as _CU
    _libm = _C.CDLL(_CU.find_library("m") or "libm.so.6")
    _libm.lgamma.restype = _C.c_double
    _libm.lgamma.argtypes = [_C.c_double]
    _lgamma = _libm.lgamma
except OSError:  # pragma: no cover
    _lgamma = math.lgamma


def sbbf_fpp(a: float) -> float:
    """model.cpp:78-103, same arithmetic in the same order (Poisson mixture of
    the per-count block rate, with the reference's Chernoff tail cut-off), so
    the sizing below picks the reference's bucket counts exactly."""
    if not math.isfinite(a) or a < 0.0:
        raise ValueError("per-block density a must be finite and nonnegative")
    if a > 1e6:
        raise ValueError("per-block density a is beyond the model's sanity bound")
    if a == 0.0:
        return 0.0
    log_a = math.log(a)
    cap = int(math.ceil(a + 40.0 * math.sqrt(a) + 64.0))
    total = 0.0
    keep = 1.0
    for i in range(cap + 1):
        di = float(i)
        log_pmf = di * log_a - a - _lgamma(di + 1.0)
        one = 1.0 - keep
        r = one * one
        r *= r
        total += math.exp(log_pmf) * (r * r)
        keep *= 31.0 / 32.0
        if di > a and total > 0.0:
            log_tail = di - a - di * math.log(di / a)
            if log_tail < math.log(1e-12 * total):
                break
    return min(total, 1.0)


def solve_a_for_fpp(target: float) -> float:
    """model.cpp:170-184 — bisection on a."""
    if not math.isfinite(target) or target <= 0.0 or target >= 1.0:
        raise ValueError("target_fpp must lie strictly between 0 and 1")
    lo, hi = 1e-3, 1e3
    while hi - lo > 1e-9:
        mid = 0.5 * (lo + hi)
        if sbbf_fpp(mid) < target:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def size_for(ndv: int, target_fpp: float) -> int:
    """model.cpp:187-212 — smallest bucket count meeting target_fpp."""
    if ndv < 1:
        raise ValueError("ndv must be at least 1")
    a = solve_a_for_fpp(target_fpp)
    n = float(ndv)
    buckets = max(1, int(math.ceil(n / a)))
    while sbbf_fpp(n / buckets) > target_fpp:
        buckets += 1
    while buckets > 1 and sbbf_fpp(n / (buckets - 1)) <= target_fpp:
        buckets -= 1
    return buckets


def read_key_lines(path: str) -> list[bytes]:
    """harness.cpp:247-260 (std::getline semantics)."""
    with open(path, "rb") as fh:
        data = fh.read()
    if not data:
        return []
    parts = data.split(b"\n")
    if data.endswith(b"\n"):
        parts.pop()
    return parts


def run_build(key_file: str, out_file: str, target_fpp: float, device: int = 0) -> dict:
    """harness.cpp:262-283: hash every line, size for the distinct count, insert, save."""
    import torch
    keys = read_key_lines(key_file)
    hashes = hash_keys(keys, 0, device) if keys else torch.zeros(0, dtype=torch.int64,
                                                                 device=torch.device("cuda", device))
    distinct = int(torch.unique(hashes).numel())
    buckets = size_for(max(1, distinct), target_fpp)
    f = SplitBlockFilter(buckets, hasher_id=KHASHER_XXH64, device=device)
    f.add_hashes(hashes)
    f.save(out_file)
    return {"keys_read": len(keys), "distinct_hashes": distinct, "num_buckets": buckets,
            "bytes": buckets * 32, "predicted_fpp": sbbf_fpp(max(1, distinct) / buckets)}


def run_query(filter_file: str, key_file: str, out=sys.stdout, device: int = 0) -> dict:
    """harness.cpp:285-304: one line per key, "maybe" or "absent"."""
    f = SplitBlockFilter.load(filter_file, device)
    if f.hasher_id() != KHASHER_XXH64:
        raise ValueError(f"filter {filter_file} was built with hasher id {f.hasher_id()}; this tool "
                         "queries with hasher id 1 (bundled XXH64)")
    keys = read_key_lines(key_file)
    if not keys:
        return {"keys": 0, "maybe": 0}
    res = f.find_hashes(hash_keys(keys, 0, device)).cpu().numpy().astype(bool)
    out.write("".join("maybe\n" if r else "absent\n" for r in res))
    return {"keys": len(keys), "maybe": int(np.count_nonzero(res))}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="sbbf-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("build")
    b.add_argument("keys")
    b.add_argument("out")
    b.add_argument("--fpp", type=float, default=0.01)
    q = sub.add_parser("query")
    q.add_argument("filter")
    q.add_argument("keys")
    args = ap.parse_args(argv)
    if args.cmd == "build":
        r = run_build(args.keys, args.out, args.fpp)
        print(f"built {r['num_buckets']} buckets ({r['bytes']} bytes) for {r['distinct_hashes']} distinct "
              f"of {r['keys_read']} keys, predicted fpp {r['predicted_fpp']:.6g}", file=sys.stderr)
    else:
        run_query(args.filter, args.keys)
    return 0


if __name__ == "__main__":
    sys.exit(main())
