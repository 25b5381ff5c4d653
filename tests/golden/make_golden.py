"""Generate tests/golden/ fixtures by running the REFERENCE itself.

Runs the unmodified reference core (oracle/_ref/libsbbf_ref.so, compiled from
/root/reference/proj/core/src by oracle/Makefile) on seeded inputs and writes
its outputs as small fixtures. Only runnable where /root/reference exists;
the committed fixtures travel to the GPU box, the reference does not.

    python tests/golden/make_golden.py            # configs 1-3 + unit cases
    python tests/golden/make_golden.py --cfg4     # also config 4 (~minutes)
    python tests/golden/make_golden.py --cfg5     # config 5 (8 GiB, 8e9 + 8e9; ~10 min)
                                                  # and the sharded bench's per-world samples

Inputs: the reference tests' own std::mt19937_64 draws (seeds from
filter_test.cpp / persist_test.cpp / acceptance.cpp) and the BASELINE.json
config streams (paper_2101_01719_b200.workload, restated on the host by the
oracle).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Oracle, Reference  # noqa: E402
from paper_2101_01719_b200 import workload as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def image_crc(img: bytes) -> int:
    return int.from_bytes(img[-4:], "little")


def unit_cases(ref: Reference, orc: Oracle) -> dict:
    g: dict = {}
    # block_index vs the big-integer oracle (filter_test.cpp:35-49 inputs).
    buckets = [1, 2, 3, 7, 4096, 1000, 999983, 1 << 20, (1 << 40) + 17, (1 << 33) + 9]
    hs = ref.mt19937_64(0x5EED0001, 2000)
    g["block_index"] = {
        "hash_seed": 0x5EED0001, "n": 2000, "buckets": buckets,
        "expected": [[ref.block_index(int(h), b) for b in buckets] for h in hs],
    }
    # make_mask (filter_test.cpp:102-114 inputs)
    hs = ref.mt19937_64(0x5EED0003, 2000)
    g["make_mask"] = {"hash_seed": 0x5EED0003, "n": 2000,
                      "expected": [ref.make_mask(int(h)) for h in hs]}
    # Filters built by the reference: (buckets, adds, insert seed, probe count)
    cases = [
        ("one_bucket_24", 1, 24, 0x5EED000A, 4096),
        ("add_then_find_57", 57, 1000, 0x5EED0004, 1000),
        ("bulk_97", 97, 1000, 0x5EED0005, 1000),
        ("monotone_11", 11, 200, 0x5EED0006, 500),
        ("backend_identity_4096", 4096, 100_000, 0x5EED0007, 10_000),
        ("instrumented_1000", 1000, 5000, 0x5EED0008, 5000),
        ("persist_512", 512, 20_000, 0xABCD01, 5000),
        ("nonpow2_7919", 7919, 200_000, 0xACC0002, 100_000),
        ("nonpow2_999983", 999_983, 3_000_000, 0xACC0009, 1_000_000),
        ("acceptance_7", 7, 1_000_000, 0xACC0001, 10_000),
    ]
    fl = []
    for name, nb, adds, seed, nprobe in cases:
        draws = ref.mt19937_64(seed, adds + nprobe)
        ins = draws[:adds]
        # probes: half inserted keys, half fresh draws
        half = min(adds, nprobe // 2)
        probes = np.concatenate([ins[:half], draws[adds: adds + nprobe - half]])
        f = ref.filter(nb)
        f.add_hashes(ins)
        res = f.find_hashes(probes)
        img = f.serialize()
        entry = {"name": name, "buckets": nb, "adds": adds, "seed": seed, "probes": int(probes.size),
                 "image_crc": image_crc(img), "popcount": orc.popcount(f.blocks()),
                 "blocks_sha256": sha(f.blocks()), "results_sha256": sha(res),
                 "hits": int(res.sum())}
        if nb <= 128:
            entry["image_hex"] = img.hex()
        fl.append(entry)
    g["filters"] = fl
    return g


def config_golden(ref: Reference, orc: Oracle, cid: int, threads: int) -> dict:
    cfg = W.CONFIGS[cid]
    t0 = time.time()
    table = W.zipf_cdf_table(cfg.inserts.zipf_s, cfg.inserts.zipf_n) if cfg.inserts.dup_num else None
    st = orc.stream(cfg.inserts, table)
    f = ref.filter(cfg.num_buckets)
    chunk = 1 << 26
    N = cfg.inserts.n
    first_ins = None
    for s in range(0, N, chunk):
        a = orc.gen_inserts(st, s, min(chunk, N - s))
        if first_ins is None:
            first_ins = [int(x) for x in a[:4]]
        f.add_hashes(a)
    img = f.serialize()
    blocks = f.blocks()
    L = cfg.lookups.n
    hits = 0
    member_hits = 0
    nonmember_hits = 0
    crc_state = 0
    first_look = None
    res_crcs = []
    for s in range(0, L, chunk):
        m = min(chunk, L - s)
        q = orc.gen_lookups(st, cfg.lookups, N, s, m)
        if first_look is None:
            first_look = [int(x) for x in q[:4]]
        r = f.find_hashes(q, threads)
        hits += int(r.sum())
        # member mask for this chunk
        j = np.arange(s, s + m, dtype=np.uint64)
        if cfg.lookups.members_first:
            mem = j < N
        else:
            p, qq = cfg.lookups.p, cfg.lookups.q
            mem = ((j + 1) * p // qq) > (j * p // qq)
        member_hits += int(r[mem].sum())
        nonmember_hits += int(r[~mem].sum())
        res_crcs.append(orc.crc32(np.packbits(r, bitorder="little").tobytes()))
    n_members = W.member_count(cfg.lookups, N, 0, L)
    out = {
        "config": cid, "num_buckets": cfg.num_buckets, "inserts": N, "lookups": L,
        "first_inserts": first_ins, "first_lookups": first_look,
        "image_crc": image_crc(img), "popcount": orc.popcount(blocks),
        "members": n_members, "member_hits": member_hits,
        "nonmembers": L - n_members, "false_positives": nonmember_hits,
        "lookup_bitmap_chunk_crcs": res_crcs, "chunk_keys": chunk,
        "seconds": round(time.time() - t0, 1),
    }
    print(f"cfg{cid}: crc={out['image_crc']:#x} fp={nonmember_hits}/{L - n_members} "
          f"members={member_hits}/{n_members} ({out['seconds']} s)", flush=True)
    return out


def image_crc_of_blocks(blocks: np.ndarray, num_buckets: int, hasher_id: int = 0) -> int:
    """FilterImage v1 trailer CRC (persist.cpp:72-88) without materialising
    the image: zlib's IEEE CRC-32 over the 17-byte header, then the blocks
    (checked against the reference's own serialize() on the smaller cases)."""
    import zlib
    hdr = b"SBBF" + bytes([1]) + hasher_id.to_bytes(4, "little") + num_buckets.to_bytes(8, "little")
    return zlib.crc32(memoryview(np.ascontiguousarray(blocks)).cast("B"), zlib.crc32(hdr)) & 0xFFFFFFFF


def stream_golden(ref: Reference, orc: Oracle, num_buckets: int, ins_spec, lk, n_ins: int, n_look: int,
                  threads: int, chunk: int = 1 << 26, serialize_check: bool = False) -> dict:
    """Insert positions [0, n_ins) of ins_spec into a reference filter of
    num_buckets in chunks (add_hashes, filter.cpp:184-190), then look up
    positions [0, n_look) of lk's mixed stream (members drawn from the n_ins
    inserts) with find_hashes over `threads` jthreads (harness.cpp:173-200).
    Large configs stream both sides in chunks (no 64 GB arrays)."""
    t0 = time.time()
    st = orc.stream(ins_spec)
    f = ref.filter(num_buckets)
    first_ins = None
    for s in range(0, n_ins, chunk):
        a = orc.gen_inserts(st, s, min(chunk, n_ins - s))
        if first_ins is None:
            first_ins = [int(x) for x in a[:4]]
        f.add_hashes(a)
    t_ins = time.time() - t0
    blocks = f.blocks()
    crc = image_crc_of_blocks(blocks, num_buckets)
    if serialize_check:
        assert crc == image_crc(f.serialize()), "zlib image CRC != reference serialize()"
    pop = orc.popcount(blocks)
    del blocks
    member_hits = nonmember_hits = 0
    res_crcs = []
    first_look = None
    for s in range(0, n_look, chunk):
        m = min(chunk, n_look - s)
        q = orc.gen_lookups(st, lk, n_ins, s, m)
        if first_look is None:
            first_look = [int(x) for x in q[:4]]
        r = f.find_hashes(q, threads)
        j = np.arange(s, s + m, dtype=np.uint64)
        mem = ((j + 1) * lk.p // lk.q) > (j * lk.p // lk.q)
        member_hits += int(r[mem].sum())
        nonmember_hits += int(r[~mem].sum())
        res_crcs.append(orc.crc32(np.packbits(r, bitorder="little").tobytes()))
    n_members = W.member_count(lk, n_ins, 0, n_look)
    out = {"num_buckets": num_buckets, "inserts": n_ins, "lookups": n_look,
           "first_inserts": first_ins, "first_lookups": first_look,
           "image_crc": crc, "popcount": pop, "members": n_members, "member_hits": member_hits,
           "nonmembers": n_look - n_members, "false_positives": nonmember_hits,
           "lookup_bitmap_chunk_crcs": res_crcs, "chunk_keys": chunk,
           "seconds": round(time.time() - t0, 1), "insert_seconds": round(t_ins, 1)}
    print(f"nb={num_buckets} ins={n_ins} look={n_look}: crc={crc:#x} fp={nonmember_hits}/{n_look - n_members} "
          f"members={member_hits}/{n_members} ({out['seconds']} s)", flush=True)
    return out


def config5_golden(ref: Reference, orc: Oracle, threads: int) -> tuple[dict, dict]:
    """Config 5 in full (8 GiB filter, 8e9 inserts of splitmix64(9), 8e9
    lookups, 25 % members, non-members splitmix64(10)) and the sharded
    bench's per-step samples: at world P every rank r originates insert
    positions [r*S, (r+1)*S) and lookup positions [r*S, (r+1)*S) of the
    config-5 streams with P*S inserts (paper_2101_01719_b200/sharded.py
    bench_main), so the union over ranks is the prefix P*S of each stream."""
    cfg = W.CONFIGS[5]
    full = stream_golden(ref, orc, cfg.num_buckets, cfg.inserts, cfg.lookups, cfg.inserts.n, cfg.lookups.n,
                         threads)
    full["config"] = 5
    samples = {}
    S = 1 << 27
    for P in (1, 2, 4, 8):
        g = stream_golden(ref, orc, cfg.num_buckets, cfg.inserts, cfg.lookups, P * S, P * S, threads,
                          serialize_check=(P == 1))
        g.update({"world": P, "per_rank_keys": S})
        samples[str(P)] = g
    return full, samples


def frontend_cases(ref: Reference) -> dict:
    """XXH64 frontend (hash.cpp) and run_fpp_sim (harness.cpp:67-109) goldens."""
    g: dict = {}
    keys = ref.mt19937_64(0xF00D, 256)
    g["u64"] = {"key_seed": 0xF00D, "n": 256, "seeds": [0, 1, 20160216],
                "expected": [[int(ref.lib.ref_hash_u64_key(int(k), s)) for s in (0, 1, 20160216)]
                             for k in keys]}
    rng = np.random.default_rng(0xBEEF)
    strings = [rng.integers(0, 256, size=int(rng.integers(0, 100)), dtype=np.uint8).tobytes()
               for _ in range(64)]
    g["bytes"] = {"hex": [s.hex() for s in strings],
                  "expected": [ref.hash_key(s, 7) for s in strings], "seed": 7}
    # acceptance.cpp:168-181,354-366 (criteria 4a-4c) and the README example
    runs = []
    for ndv, nbytes, seed in ((100_000, 131_072, 20160216), (1_000_000, 1_048_576, 20160216),
                              (100_000_000, 134_217_728, 20160216), (100_000, 131_072, 1)):
        fp, crc = ref.fpp_sim(ndv, nbytes, 1_000_000, seed)
        runs.append({"ndv": ndv, "filter_bytes": nbytes, "queries": 1_000_000, "seed": seed,
                     "false_positives": fp, "image_crc": crc})
        print(f"fpp-sim ndv={ndv} bytes={nbytes} seed={seed}: fp={fp} crc={crc:#x}", flush=True)
    g["fpp_sim"] = runs
    # sbbf build / query (harness.cpp:262-304) on a deterministic key file
    keys, probes = build_query_inputs()
    hashes = np.array([ref.hash_key(k, 0) for k in keys], np.uint64)
    distinct = int(np.unique(hashes).size)
    g_build = {}
    for fpp in (0.01, 0.001, 0.2):
        nb = int(ref.lib.ref_size_for(max(1, distinct), fpp))
        f = ref.filter(nb, 1)
        f.add_hashes(hashes)
        ph = np.array([ref.hash_key(k, 0) for k in probes], np.uint64)
        res = f.find_hashes(ph)
        g_build[str(fpp)] = {"num_buckets": nb, "image_crc": image_crc(f.serialize()),
                             "maybe": int(res.sum()), "answers_sha256": sha(res)}
    g["build_query"] = {"keys_read": len(keys), "distinct": distinct, "runs": g_build}
    return g


def build_query_inputs():
    """Key file lines for the build/query golden: 20k keys with duplicates
    and an empty line; probes = every other key plus absent ones."""
    keys = [f"key-{i}".encode() for i in range(20_000)] + [f"key-{i}".encode() for i in range(0, 20_000, 7)]
    keys.append(b"")
    probes = keys[::2] + [f"absent-{i}".encode() for i in range(30_000)]
    return keys, probes


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg4", action="store_true")
    ap.add_argument("--cfg5", action="store_true")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    ref, orc = Reference(), Oracle()
    if args.cfg5:
        full, samples = config5_golden(ref, orc, args.threads)
        with open(os.path.join(OUT, "config5.json"), "w") as fh:
            json.dump({"5": full, "samples": samples}, fh, indent=1)
        return
    with open(os.path.join(OUT, "unit_cases.json"), "w") as fh:
        json.dump(unit_cases(ref, orc), fh)
    with open(os.path.join(OUT, "frontend.json"), "w") as fh:
        json.dump(frontend_cases(ref), fh)
    cfgs = {}
    path = os.path.join(OUT, "configs.json")
    if os.path.exists(path):
        with open(path) as fh:
            cfgs = json.load(fh)
    for cid in (1, 2, 3) + ((4,) if args.cfg4 else ()):
        cfgs[str(cid)] = config_golden(ref, orc, cid, args.threads)
    with open(path, "w") as fh:
        json.dump(cfgs, fh, indent=1)


if __name__ == "__main__":
    main()
