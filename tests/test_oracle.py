"""CPU: pin the oracle (oracle/sbbf_oracle.c) before trusting it.

1. The reference's own known-answer vectors, transcribed from its tests
   (paths relative to /root/reference/proj/).
2. The golden fixtures produced by running the reference itself
   (tests/golden/make_golden.py over oracle/_ref).
3. Direct differential runs against oracle/_ref where it is built.
"""
import hashlib
import os

import numpy as np
import pytest

from oracle import LANE_SEEDS, bits_to_bytes
from paper_2101_01719_b200 import workload as W


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# --- filter_test.cpp:22-33 ----------------------------------------------------
BLOCK_INDEX_KAT = [
    (0, 12345, 0),
    (1 << 63, 4, 2),
    (0xDEADBEEFDEADBEEF, 1000, 869),
    (0xA00641A9F1E54A8B, 7919, 4950),
    (0xC693565F940AF963, 7919, 6142),
    (0x39A72DABD56A2742, 7919, 1783),
    (0xDFA132D748FA2734, 7919, 6917),
    (0xFFFFFFFFFFFFFFFF, 1, 0),
    (0xFFFFFFFFFFFFFFFF, 1000, 999),
]

# --- filter_test.cpp:90-99 ----------------------------------------------------
MASK_KAT = {
    0xDEADBEEFDEADBEEF: [0x00008000, 0x20000000, 0x00004000, 0x00001000,
                         0x02000000, 0x00002000, 0x00200000, 0x01000000],
    0x0123456789ABCDEF: [0x00080000, 0x00040000, 0x00800000, 0x40000000,
                         0x00010000, 0x00000010, 0x01000000, 0x00001000],
}


def test_block_index_kat(oracle):
    for h, nb, want in BLOCK_INDEX_KAT:
        assert oracle.block_index(h, nb) == want


def test_make_mask_kat(oracle):
    assert oracle.make_mask(0) == [1] * 8                       # filter_test.cpp:67-72
    want_bits = [8, 8, 20, 17, 5, 14, 11, 19]                   # filter_test.cpp:73-80
    assert want_bits == [s >> 27 for s in LANE_SEEDS]
    assert oracle.make_mask(1) == [1 << b for b in want_bits]
    assert oracle.make_mask(0xFFFFFFFF00000000) == [1] * 8      # filter_test.cpp:81-89
    assert oracle.make_mask(0x00000000DEADBEEF) == oracle.make_mask(0x12345678DEADBEEF)
    for h, lanes in MASK_KAT.items():
        assert oracle.make_mask(h) == lanes


def test_add_hash_zero_one_bucket(oracle):
    b = oracle.build(1, [0])                                    # filter_test.cpp:164-170
    assert b.tolist() == [[1] * 8]


def test_crc_check_value(oracle):
    assert oracle.crc32(b"123456789") == 0xCBF43926             # persist_test.cpp:42-47
    assert oracle.crc32(b"") == 0


def test_empty_image_layout(oracle):
    img = oracle.serialize(oracle.new_blocks(1))                # persist_test.cpp:49-70
    assert len(img) == 53
    assert img[:4] == b"SBBF" and img[4] == 1
    assert img[5:9] == b"\0\0\0\0" and int.from_bytes(img[9:17], "little") == 1
    assert img[17:49] == b"\0" * 32


def test_one_hash_changes_eight_bytes(oracle):
    h = 0x9E3779B97F4A7C15                                      # persist_test.cpp:81-111
    before = oracle.serialize(oracle.new_blocks(4))
    after = oracle.serialize(oracle.build(4, [h]))
    blk = oracle.block_index(h, 4)
    expected = set()
    for lane, seed in enumerate(LANE_SEEDS):
        bit = ((seed * (h & 0xFFFFFFFF)) & 0xFFFFFFFF) >> 27
        expected.add(17 + blk * 32 + lane * 4 + bit // 8)
    diffs = {i for i in range(len(before) - 4) if before[i] != after[i]}
    assert diffs == expected and len(expected) == 8
    assert before[-4:] != after[-4:]


def test_deserialize_errors(oracle):
    img = bytearray(oracle.serialize(oracle.build(3, [1, 2, 3])))
    rc, blocks, hid = oracle.deserialize(bytes(img))
    assert rc == 0 and blocks.shape == (3, 8) and hid == 0
    assert oracle.deserialize(bytes(img[:20]))[0] == 1         # kTruncated
    assert oracle.deserialize(bytes(img[:-1]))[0] == 1
    bad = bytearray(img); bad[0] = ord("X")
    assert oracle.deserialize(bytes(bad))[0] == 2               # kBadMagic
    bad = bytearray(img); bad[4] = 2
    assert oracle.deserialize(bytes(bad))[0] == 3               # kBadVersion
    zero = bytearray(oracle.serialize(oracle.new_blocks(1)))
    zero[9:17] = b"\0" * 8
    assert oracle.deserialize(bytes(zero))[0] == 4              # kBadBucketCount
    bad = bytearray(img); bad[-1] ^= 1
    assert oracle.deserialize(bytes(bad))[0] == 5               # kBadChecksum


def test_xxh64_vectors(oracle):
    # hash_test.cpp:36-96 (pattern bytes i*31+7)
    pat = lambda n: bytes(((i * 31 + 7) & 0xFF) for i in range(n))  # noqa: E731
    vec = [(0, 0, 0xEF46DB3751D8E999), (1, 0, 0xA96C7F0CE858BBB7), (3, 1, 0x598AFE4FBB09D9F6),
           (8, 0x9E3779B97F4A7C15, 0x758848F033FA76A2), (32, 0, 0x8D57D6A4671CC43D),
           (33, 1, 0xB1575979B72C805A), (100, 0x9E3779B97F4A7C15, 0xBC7AB33BE7528C18)]
    for n, seed, want in vec:
        assert oracle.xxh64(pat(n), seed) == want
    assert oracle.xxh64(b"a", 0) == 0xD24EC4F1A98C6E5B
    assert oracle.xxh64(b"hello world", 42) == 0x69C2B68F9D9352A1


def test_mt19937_64_matches_std(oracle):
    # The C++ standard pins the 10000th output of default-seeded mt19937_64.
    assert int(oracle.mt19937_64(5489, 10000)[-1]) == 9981545732273789042


# --- golden fixtures made by the reference ---------------------------------------
def test_golden_block_index(oracle, golden_units):
    g = golden_units["block_index"]
    hs = oracle.mt19937_64(g["hash_seed"], g["n"])
    for h, row in zip(hs[:400], g["expected"][:400]):
        assert [oracle.block_index(int(h), b) for b in g["buckets"]] == row


def test_golden_make_mask(oracle, golden_units):
    g = golden_units["make_mask"]
    hs = oracle.mt19937_64(g["hash_seed"], g["n"])
    for h, row in zip(hs[:500], g["expected"][:500]):
        assert oracle.make_mask(int(h)) == row


@pytest.mark.parametrize("idx", range(10))
def test_golden_filters(oracle, golden_units, idx):
    c = golden_units["filters"][idx]
    draws = oracle.mt19937_64(c["seed"], c["adds"] + c["probes"])
    ins = draws[: c["adds"]]
    half = min(c["adds"], c["probes"] // 2)
    probes = np.concatenate([ins[:half], draws[c["adds"]: c["adds"] + c["probes"] - half]])
    b = oracle.build(c["buckets"], ins)
    assert sha(b) == c["blocks_sha256"]
    assert oracle.image_crc(b) == c["image_crc"]
    assert oracle.popcount(b) == c["popcount"]
    res = oracle.find_hashes(b, probes, threads=4)
    assert sha(res) == c["results_sha256"] and int(res.sum()) == c["hits"]
    assert np.array_equal(bits_to_bytes(oracle.find_bits(b, probes), probes.size), res)
    if "image_hex" in c:
        assert oracle.serialize(b).hex() == c["image_hex"]


@pytest.mark.parametrize("cid", [1, 2] + ([3] if os.environ.get("SBBF_SLOW") else []))
def test_golden_configs(oracle, golden_configs, cid):
    g = golden_configs[str(cid)]
    cfg = W.CONFIGS[cid]
    st = oracle.stream(cfg.inserts)
    ins = oracle.gen_inserts(st, 0, cfg.inserts.n)
    assert [int(x) for x in ins[:4]] == g["first_inserts"]
    b = oracle.build(cfg.num_buckets, ins)
    assert oracle.image_crc(b) == g["image_crc"]
    assert oracle.popcount(b) == g["popcount"]
    look = oracle.gen_lookups(st, cfg.lookups, cfg.inserts.n, 0, cfg.lookups.n)
    assert [int(x) for x in look[:4]] == g["first_lookups"]
    res = oracle.find_hashes(b, look, threads=8)
    chunk = g["chunk_keys"]
    crcs = [oracle.crc32(np.packbits(res[s:s + chunk], bitorder="little").tobytes())
            for s in range(0, res.size, chunk)]
    assert crcs == g["lookup_bitmap_chunk_crcs"]


def test_survey_golden_values(golden_configs):
    # values the survey computed with the reference.
    assert golden_configs["1"]["image_crc"] == 0xE34F8BEF
    assert golden_configs["1"]["false_positives"] == 10190
    assert golden_configs["1"]["first_inserts"][:3] == [0x910A2DEC89025CC1, 0xBEEB8DA1658EEC67,
                                                        0xF893A2EEFB32555E]
    assert golden_configs["2"]["image_crc"] == 0x666876BF
    assert golden_configs["2"]["false_positives"] == 135978
    assert golden_configs["3"]["image_crc"] == 0xDE283BC7
    assert golden_configs["3"]["false_positives"] == 8224912
    for k in ("1", "2", "3"):
        assert golden_configs[k]["member_hits"] == golden_configs[k]["members"]  # no false negatives


# --- direct differential against the reference (where oracle/_ref exists) ------
def test_oracle_vs_reference_random(oracle, reference):
    rng = np.random.default_rng(7)
    for nb in (1, 2, 7, 57, 4096, 999983):
        hs = rng.integers(0, 2**64, size=20000, dtype=np.uint64)
        assert np.array_equal(oracle.build(nb, hs), reference.build(nb, hs))
        f = reference.filter(nb)
        f.add_hashes(hs[:10000])
        assert np.array_equal(oracle.find_hashes(f.blocks(), hs), f.find_hashes(hs))
    for h in rng.integers(0, 2**64, size=200, dtype=np.uint64):
        assert oracle.make_mask(int(h)) == reference.make_mask(int(h))
        for nb in (3, 1000, (1 << 40) + 17):
            assert oracle.block_index(int(h), nb) == reference.block_index(int(h), nb)


def test_oracle_image_vs_reference(oracle, reference):
    hs = oracle.mt19937_64(0xABCD01, 20000)
    f = reference.filter(512)
    f.add_hashes(hs)
    img = f.serialize()
    assert oracle.serialize(f.blocks()) == img
    rc, blocks, hid = oracle.deserialize(img)
    assert rc == 0 and np.array_equal(blocks, f.blocks())
    bad = bytearray(img); bad[-1] ^= 1
    assert reference.deserialize_code(bytes(bad)) == oracle.deserialize(bytes(bad))[0] == 5


def test_xxh64_vs_reference(oracle, reference):
    rng = np.random.default_rng(3)
    for n in list(range(0, 70)) + [100, 1000]:
        data = rng.integers(0, 256, size=n, dtype=np.uint8).tobytes()
        for seed in (0, 1, 0x9E3779B97F4A7C15):
            assert oracle.xxh64(data, seed) == reference.hash_key(data, seed)
