"""The reference's ``sbbf`` toolkit commands on the GPU (tools/main.cpp,
tools/harness.cpp): ``build`` / ``query`` from key files (harness.cpp:247-304),
``fpp-sim`` (run_fpp_sim, harness.cpp:67-109), ``bench`` (run_bench,
harness.cpp:132-245), ``size`` (model.cpp:187-212) and ``model``
(run_model, harness.cpp:110-129), with the model they use (model.cpp:78-236)
restated bit-exactly.

    python -m paper_2101_01719_b200.tools build KEYS OUT.sbbf --fpp 0.01
    python -m paper_2101_01719_b200.tools query OUT.sbbf KEYS      # maybe/absent per line
    python -m paper_2101_01719_b200.tools fpp-sim --ndv 1000000 --bytes 1048576 [--key-mode strings]
    python -m paper_2101_01719_b200.tools bench --ndv 1000000 --bytes 1048576
    python -m paper_2101_01719_b200.tools size --ndv 1000000 --fpp 0.01

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

from .filter import PersistError, SplitBlockFilter, hash_keys

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


EFFICIENT_FPP_MIN, EFFICIENT_FPP_MAX = 0.004, 0.19   # model.hpp:11-12


def sizing(ndv: int, target_fpp: float) -> dict:
    """model.cpp:187-212 SizingResult."""
    if not (math.isfinite(target_fpp) and 0.0 < target_fpp < 1.0):
        raise ValueError("target_fpp must lie strictly between 0 and 1")
    buckets = size_for(ndv, target_fpp)
    a = ndv / buckets
    return {"num_buckets": buckets, "bytes": buckets * 32, "a": a, "predicted_fpp": sbbf_fpp(a),
            "outside_efficient_range": target_fpp < EFFICIENT_FPP_MIN or target_fpp > EFFICIENT_FPP_MAX}


WITHIN_2X_BOUND = 2.1   # harness.hpp:55


def standard_bloom_fpp(bits_per_key: float, k: int) -> float:
    """model.cpp:130-140."""
    if not math.isfinite(bits_per_key) or bits_per_key <= 0.0:
        raise ValueError("bits_per_key must be positive")
    if k < 1:
        raise ValueError("k must be at least 1")
    return math.pow(1.0 - math.exp(-float(k) / bits_per_key), float(k))


def optimal_bloom_k(bits_per_key: float) -> int:
    """model.cpp:142-158: best integer k over 1..max(16, ceil(bpk*ln2)+2)."""
    if not math.isfinite(bits_per_key) or bits_per_key <= 0.0:
        raise ValueError("bits_per_key must be positive")
    k_max = max(16, int(math.ceil(bits_per_key * math.log(2))) + 2)
    best_k, best = 1, standard_bloom_fpp(bits_per_key, 1)
    for k in range(2, k_max + 1):
        f = standard_bloom_fpp(bits_per_key, k)
        if f < best:
            best, best_k = f, k
    return best_k


def run_model(a_min: float = 20.0, a_max: float = 52.0, steps: int = 65) -> dict:
    """run_model + within_2x_report (harness.cpp:110-129, model.cpp:214-236):
    the sbbf fpp against a same-space standard Bloom filter (optimal k)."""
    if not (a_min >= 0.0) or a_min > a_max:
        raise ValueError("--a-min must satisfy 0 <= a-min <= a-max")
    if steps < 1:
        raise ValueError("--steps must be at least 1")
    if steps == 1 and a_min != a_max:
        raise ValueError("--steps 1 needs --a-min equal to --a-max")
    rows, max_ratio = [], 0.0
    for i in range(steps):
        t = 0.0 if steps == 1 else i / (steps - 1)
        a = a_min + t * (a_max - a_min)
        row = {"a": a, "bits_per_key": 0.0, "sbbf_fpp": 0.0, "standard_fpp": 0.0, "ratio": 0.0}
        if a > 0.0:
            bpk = 256.0 / a
            sb = sbbf_fpp(a)
            st = standard_bloom_fpp(bpk, optimal_bloom_k(bpk))
            row.update(bits_per_key=bpk, sbbf_fpp=sb, standard_fpp=st, ratio=sb / st)
            max_ratio = max(max_ratio, row["ratio"])
        rows.append(row)
    return {"rows": rows, "max_ratio": max_ratio}


def run_bench(ndv: int, filter_bytes: int, seed: int = 1, reps: int = 5, huge_ok: bool = False,
              device: int = 0) -> dict:
    """run_bench (harness.cpp:132-245) on the GPU: hashes of the counters
    [0, ndv) pre-generated on the device, then `reps` fresh-filter inserts and
    full lookups, device-timed (median); every inserted key must be found;
    the fpp columns come from 100,000 negative probes."""
    import statistics

    import torch

    from .fppsim import HUGE_NDV_THRESHOLD, NEGATIVE_COUNTER_BASE
    from .filter import hash_u64_keys
    if ndv > NEGATIVE_COUNTER_BASE:
        raise ValueError("--ndv must not exceed 2^32 (the negative-query key space starts there)")
    if ndv > HUGE_NDV_THRESHOLD and not huge_ok:
        raise ValueError("--ndv beyond 10M is paper scale; pass --huge to allow it")
    if reps < 3:
        raise ValueError("--reps must be at least 3")
    if ndv < 1:
        raise ValueError("--ndv must be positive")
    if filter_bytes < 32:
        raise ValueError("--bytes must be at least 32 (one block)")
    buckets = filter_bytes // 32
    dev = torch.device("cuda", device)
    hashes = hash_u64_keys(torch.arange(ndv, dtype=torch.int64, device=dev), seed)
    results = torch.empty(ndv, dtype=torch.uint8, device=dev)
    f = SplitBlockFilter(buckets, hasher_id=KHASHER_XXH64, device=device)
    ti, tl = [], []
    for _ in range(reps):
        f.clear()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        f.add_hashes(hashes)
        e[1].record()
        f.find_hashes(hashes, results)
        e[2].record()
        torch.cuda.synchronize(dev)
        ti.append(e[0].elapsed_time(e[1]) * 1e-3)
        tl.append(e[1].elapsed_time(e[2]) * 1e-3)
    found = int(results.sum(dtype=torch.int64).item())
    if found != ndv:
        raise RuntimeError("benchmark lookups lost inserted keys")
    probes = hash_u64_keys(torch.arange(NEGATIVE_COUNTER_BASE, NEGATIVE_COUNTER_BASE + 100_000,
                                        dtype=torch.int64, device=dev), seed)
    fpp = int(f.find_hashes(probes).sum(dtype=torch.int64).item()) / 100_000
    model = sbbf_fpp(ndv / buckets)
    base = {"ndv": ndv, "filter_bytes": buckets * 32, "threads": 1, "measured_fpp": fpp, "model_fpp": model}
    ins = dict(base, op="insert", wall_time_s=statistics.median(ti))
    look = dict(base, op="lookup", wall_time_s=statistics.median(tl))
    for r in (ins, look):
        r["million_ops_per_sec"] = ndv / r["wall_time_s"] / 1e6
    return {"insert": ins, "lookup": look, "device": torch.cuda.get_device_name(dev)}


def _print_report(r: dict) -> None:
    """main.cpp print_report format."""
    print(f"{r['op']:<8} ndv={r['ndv']} bytes={r['filter_bytes']} threads={r['threads']} "
          f"rate={r['million_ops_per_sec']:.1f} M/s measured_fpp={r['measured_fpp']:.6f} "
          f"model_fpp={r['model_fpp']:.6f} wall={r['wall_time_s']:.3f}s")


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
    """Exit codes as main.cpp: 0 ok, 1 usage, 2 I/O."""
    import json

    ap = argparse.ArgumentParser(prog="sbbf-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("build", help="hash a newline-delimited key file into a filter image")
    b.add_argument("keys")
    b.add_argument("out")
    b.add_argument("--fpp", type=float, default=0.01)
    q = sub.add_parser("query", help="print maybe/absent for each key in a file ('absent' is definitive)")
    q.add_argument("filter")
    q.add_argument("keys")
    fs = sub.add_parser("fpp-sim", help="insert ndv keys, probe disjoint keys, compare measured vs model fpp")
    fs.add_argument("--ndv", type=int, required=True)
    fs.add_argument("--bytes", type=int)
    fs.add_argument("--fpp", type=float)
    fs.add_argument("--queries", type=int, default=1_000_000)
    fs.add_argument("--seed", type=int, default=1)
    fs.add_argument("--key-mode", default="random64")
    fs.add_argument("--huge", action="store_true")
    fs.add_argument("--json", action="store_true")
    md = sub.add_parser("model", help="tabulate sbbf fpp against a same-space standard Bloom filter")
    md.add_argument("--a-min", type=float, default=20.0)
    md.add_argument("--a-max", type=float, default=52.0)
    md.add_argument("--steps", type=int, default=65)
    md.add_argument("--csv")
    md.add_argument("--json", action="store_true")
    md.add_argument("--assert-2x", action="store_true")
    sz = sub.add_parser("size", help="smallest filter meeting a target fpp")
    sz.add_argument("--ndv", type=int, required=True)
    sz.add_argument("--fpp", type=float, required=True)
    sz.add_argument("--json", action="store_true")
    bn = sub.add_parser("bench", help="time bulk insert and lookup over pre-generated hashes (GPU)")
    bn.add_argument("--ndv", type=int, required=True)
    bn.add_argument("--bytes", type=int, required=True)
    bn.add_argument("--seed", type=int, default=1)
    bn.add_argument("--reps", type=int, default=5)
    bn.add_argument("--huge", action="store_true")
    bn.add_argument("--json", action="store_true")
    args = ap.parse_args(argv)
    try:
        if args.cmd == "build":
            r = run_build(args.keys, args.out, args.fpp)
            print(f"built {r['num_buckets']} buckets ({r['bytes']} bytes) for {r['distinct_hashes']} distinct "
                  f"of {r['keys_read']} keys, predicted fpp {r['predicted_fpp']:.6g}", file=sys.stderr)
        elif args.cmd == "query":
            r = run_query(args.filter, args.keys)
            print(f"{r['keys']} keys: {r['maybe']} maybe, {r['keys'] - r['maybe']} absent", file=sys.stderr)
        elif args.cmd == "fpp-sim":
            from .fppsim import fpp_sim
            r = fpp_sim(args.ndv, args.bytes, args.queries, args.seed, huge_ok=args.huge, target_fpp=args.fpp,
                        key_mode=args.key_mode)
            r.pop("filter", None)
            r["threads"] = 1
            if args.json:
                print(json.dumps(r, indent=2))
            else:
                _print_report(r)
                ratio = r["measured_fpp"] / r["model_fpp"] if r["model_fpp"] > 0 else 0.0
                print(f"measured/model fpp ratio: {ratio:.3f}")
        elif args.cmd == "model":
            r = run_model(args.a_min, args.a_max, args.steps)
            if args.json:
                print(json.dumps(r, indent=2))
            else:
                print(f"{'a':>10} {'bits_per_key':>14} {'sbbf_fpp':>14} {'standard_fpp':>14} {'ratio':>10}")
                for row in r["rows"]:
                    print(f"{row['a']:10.3f} {row['bits_per_key']:14.4f} {row['sbbf_fpp']:14.6g} "
                          f"{row['standard_fpp']:14.6g} {row['ratio']:10.4f}")
                print(f"max ratio: {r['max_ratio']:.4f}")
            if args.csv:
                with open(args.csv, "w") as fh:
                    fh.write("a,bits_per_key,sbbf_fpp,standard_fpp,ratio\n")
                    for row in r["rows"]:
                        fh.write(",".join(f"{row[k]:.10g}" for k in
                                          ("a", "bits_per_key", "sbbf_fpp", "standard_fpp", "ratio")) + "\n")
            if args.assert_2x and r["max_ratio"] > WITHIN_2X_BOUND:
                print(f"FAIL: max sbbf/standard fpp ratio {r['max_ratio']:.4f} exceeds {WITHIN_2X_BOUND:.2f}",
                      file=sys.stderr)
                return 3
        elif args.cmd == "size":
            r = sizing(args.ndv, args.fpp)
            if args.json:
                print(json.dumps(r, indent=2))
            else:
                print(f"ndv={args.ndv} target_fpp={args.fpp:g} -> buckets={r['num_buckets']} bytes={r['bytes']} "
                      f"(a={r['a']:.3f}, predicted fpp={r['predicted_fpp']:.6f})")
            if r["outside_efficient_range"]:
                print(f"warning: target fpp {args.fpp:g} is outside the efficient range [0.4%, 19%] of the "
                      "eight-lane layout; the filter will be correct but oversized relative to other designs",
                      file=sys.stderr)
        else:
            r = run_bench(args.ndv, args.bytes, args.seed, args.reps, args.huge)
            if args.json:
                print(json.dumps(r, indent=2))
            else:
                _print_report(r["insert"])
                _print_report(r["lookup"])
    except (PersistError, OSError) as exc:  # main.cpp: PersistError -> kExitIo
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except ValueError as exc:                # UsageError / std::domain_error -> kExitUsage
        print(f"error: {exc}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
