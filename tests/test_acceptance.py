"""The reference's acceptance suite (proj/tests/acceptance/acceptance.cpp,
criteria 1-9), criterion by criterion, run against this implementation: the
GPU filter for the filter criteria, the model restatement for the analytic
ones. Thresholds and seeds are the reference's."""
import math

import numpy as np
import pytest

from paper_2101_01719_b200 import tools
from paper_2101_01719_b200.fppsim import sbbf_fpp

SEEDS = [0x44974D91, 0x47B6137B, 0xA2B7289D, 0x8824AD5B, 0x2DF1424B, 0x705495C7, 0x5C6BFB31, 0x9EFC4947]


# --- criterion 5: within 2x of a standard Bloom filter (acceptance.cpp:210-221)
def test_criterion5_within_2x():
    r = tools.run_model(20.0, 52.0, 65)
    assert len(r["rows"]) == 65 and r["max_ratio"] <= 2.1


# --- criterion 6: space comparison at one percent (acceptance.cpp:223-232)
def test_criterion6_space_comparison():
    a_star = tools.solve_a_for_fpp(0.0100)
    bpk = 256.0 / a_star
    standard = tools.standard_bloom_fpp(bpk, tools.optimal_bloom_k(bpk))
    assert 0.0056 <= standard <= 0.0070


# --- criterion 7: efficient-range endpoint rates (acceptance.cpp:234-242)
def test_criterion7_efficient_range_endpoints():
    assert 0.003 <= sbbf_fpp(20.0) <= 0.005
    assert 0.14 <= sbbf_fpp(52.0) <= 0.24


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_criterion2_bit_exact_vectors_and_path_identity(cuda, oracle):
    """acceptance.cpp:86-138: 10^4 mt19937_64(0xacc0002) hashes against the
    oracle for block_index at {1, 7, 1000, 4096, 999983, 2^33+9} buckets and
    for make_mask; every insert path byte-identical over 10^5 adds."""
    import torch

    from paper_2101_01719_b200 import SplitBlockFilter, _lib, block_index_batch, make_mask_batch
    h = oracle.mt19937_64(0xACC0002, 10_000 + 100_000)
    d = torch.from_numpy(h[:10_000].view(np.int64)).to(cuda)
    for nb in (1, 7, 1000, 4096, 999983, (1 << 33) + 9):
        got = block_index_batch(d, nb).cpu().numpy().view(np.uint64)
        want = np.array([oracle.block_index(int(x), nb) for x in h[:10_000]], np.uint64)
        assert np.array_equal(got, want), nb
    lanes = make_mask_batch(d).cpu().numpy().view(np.uint32).reshape(-1, 8)
    assert np.array_equal(lanes, np.array([oracle.make_mask(int(x)) for x in h[:10_000]], np.uint32))
    adds = torch.from_numpy(h[10_000:].view(np.int64)).to(cuda)
    images = set()
    for v in (_lib.INSERT_LANE8, _lib.INSERT_LANE8_TEST, _lib.INSERT_THREAD, _lib.INSERT_WIDE,
              _lib.INSERT_WIDE_TEST, _lib.INSERT_BLOCKED):
        f = SplitBlockFilter(4096)
        f.set_insert_variant(v)
        f.add_hashes(adds)
        images.add(bytes(f.serialize()))
    assert len(images) == 1
    assert images.pop() == oracle.serialize(oracle.build(4096, h[10_000:]))


@pytest.mark.gpu
def test_criterion3_model_vs_simulation(cuda):
    """acceptance.cpp:140-164: the series within 3 binomial SEs of the mean of
    25 Monte-Carlo replicates (4096 blocks, 10^6 queries) at a in
    {5, 20, 26, 33, 43, 52} — with the GPU Monte-Carlo oracle."""
    from paper_2101_01719_b200.fppsim import sbbf_fpp_mc
    for a in (5.0, 20.0, 26.0, 33.0, 43.0, 52.0):
        series = sbbf_fpp(a)
        mc = sum(sbbf_fpp_mc(a, 4096, 1_000_000, 0xACC0003 + 1000 * r + int(a)) for r in range(25)) / 25
        se = math.sqrt(series * (1.0 - series) / 1e6)
        assert abs(mc - series) <= 3.0 * se, (a, mc, series)


@pytest.mark.gpu
def test_criterion4d_bench_reports_wellformed(cuda):
    """acceptance.cpp:180-208: run_bench(100k keys, 131072 bytes, 3 reps)."""
    r = tools.run_bench(100_000, 131_072, 1, 3)
    for rep in (r["insert"], r["lookup"]):
        assert rep["million_ops_per_sec"] > 0 and math.isfinite(rep["million_ops_per_sec"])
        assert rep["wall_time_s"] > 0 and rep["filter_bytes"] == 131_072
        for field in ("op", "ndv", "filter_bytes", "threads", "million_ops_per_sec", "measured_fpp",
                      "model_fpp", "wall_time_s"):
            assert field in rep


@pytest.mark.gpu
def test_criterion8_persistence(cuda, oracle):
    """acceptance.cpp:244-298: round trips at {1, 2, 7, 4096} buckets with
    24 adds per bucket (hasher id 1), and distinct errors for a corrupted,
    wrong-magic, wrong-version, truncated and empty image."""
    import torch

    from paper_2101_01719_b200 import SplitBlockFilter
    from paper_2101_01719_b200.filter import PersistError
    rng = oracle.mt19937_64(0xACC0008, 200_000)
    used = 0
    for nb in (1, 2, 7, 4096):
        f = SplitBlockFilter(nb, hasher_id=1)
        h = rng[used:used + 24 * nb]
        used += 24 * nb
        f.add_hashes(torch.from_numpy(h.view(np.int64)).to(cuda))
        img = bytes(f.serialize())
        back = SplitBlockFilter.deserialize(img)
        assert back == f and bytes(back.serialize()) == img
    f = SplitBlockFilter(7, hasher_id=1)
    f.add_hashes(torch.from_numpy(rng[used:used + 100].view(np.int64)).to(cuda))
    good = bytearray(f.serialize())

    def code(b):
        with pytest.raises(PersistError) as e:
            SplitBlockFilter.deserialize(bytes(b))
        return e.value.code

    corrupted = bytearray(good)
    corrupted[17 + 11] ^= 0x10
    magic = bytearray(good)
    magic[1] = ord("X")
    version = bytearray(good)
    version[4] = 9
    codes = [code(corrupted), code(magic), code(version), code(good[:-3]), code(b"")]
    assert codes == ["kBadChecksum", "kBadMagic", "kBadVersion", "kTruncated", "kTruncated"]


@pytest.mark.gpu
def test_criterion9_one_block_eight_lanes(cuda, oracle):
    """acceptance.cpp:300-336: every add touches exactly one block and sets
    one bit per lane (the make_mask of its hash), at 1, 10^3 and 10^6
    buckets; find agrees with the reference filter."""
    from paper_2101_01719_b200 import SplitBlockFilter
    h = oracle.mt19937_64(0xACC0009, 2_000)
    for nb in (1, 1000, 1_000_000):
        f = SplitBlockFilter(nb)
        before = f.blocks().copy()
        for i in range(0, 200, 2):
            f.add_hash(int(h[i]))
            after = f.blocks()
            changed = np.nonzero(np.any(before != after, axis=1))[0]
            b = oracle.block_index(int(h[i]), nb)
            assert set(changed.tolist()) <= {b}
            assert np.array_equal(after[b], before[b] | np.array(oracle.make_mask(int(h[i])), np.uint32))
            before = after.copy()
        ref = oracle.build(nb, h[0:200:2])
        probes = h[1:200:2]
        got = [f.find_hash(int(p)) for p in probes]
        assert got == [bool(x) for x in oracle.find_hashes(ref, probes)]
