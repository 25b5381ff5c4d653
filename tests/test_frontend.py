"""XXH64 key frontend (hash.cpp) and GPU fpp-sim (harness.cpp:67-109) against
the reference's outputs (tests/golden/frontend.json, made by oracle/_ref)."""
import json
import os

import numpy as np
import pytest

from paper_2101_01719_b200.fppsim import sbbf_fpp

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "frontend.json")


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


def test_oracle_xxh64_matches_reference_golden(oracle, golden):
    g = golden["u64"]
    keys = oracle.mt19937_64(g["key_seed"], g["n"])
    for k, row in zip(keys, g["expected"]):
        assert [oracle.xxh64(int(k).to_bytes(8, "little"), s) for s in g["seeds"]] == row
    b = golden["bytes"]
    for hx, want in zip(b["hex"], b["expected"]):
        assert oracle.xxh64(bytes.fromhex(hx), b["seed"]) == want


def test_model_series():
    # model_test.cpp:33,35 — the series at configs 1 and 2 densities
    assert abs(sbbf_fpp(24.4140625) - 0.01019178249) < 1e-10
    assert abs(sbbf_fpp(30.517578125) - 0.02725598177) < 1e-10
    assert sbbf_fpp(0.0) == 0.0


def test_fppsim_argument_errors():
    from paper_2101_01719_b200.fppsim import fpp_sim
    with pytest.raises(ValueError):
        fpp_sim(10, 16)                          # < one block
    with pytest.raises(ValueError):
        fpp_sim(20_000_000, 1 << 20)             # paper scale without huge_ok
    with pytest.raises(ValueError):
        fpp_sim(10, 1 << 20, negative_queries=0)


# --------------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_device_hash_u64_and_bytes(cuda, oracle, golden):
    import torch

    from paper_2101_01719_b200.filter import hash_keys, hash_u64_keys
    g = golden["u64"]
    keys = oracle.mt19937_64(g["key_seed"], g["n"])
    d = torch.from_numpy(keys.view(np.int64)).to(cuda)
    for j, seed in enumerate(g["seeds"]):
        got = hash_u64_keys(d, seed).cpu().numpy().view(np.uint64)
        assert [int(x) for x in got] == [row[j] for row in g["expected"]]
    b = golden["bytes"]
    got = hash_keys([bytes.fromhex(h) for h in b["hex"]], b["seed"]).cpu().numpy().view(np.uint64)
    assert [int(x) for x in got] == b["expected"]
    # every tail path: lengths 0..100 against the oracle
    rng = np.random.default_rng(5)
    blobs = [rng.integers(0, 256, size=n, dtype=np.uint8).tobytes() for n in range(101)]
    got = hash_keys(blobs, 0x9E3779B97F4A7C15).cpu().numpy().view(np.uint64)
    assert [int(x) for x in got] == [oracle.xxh64(x, 0x9E3779B97F4A7C15) for x in blobs]


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 4, 5, 6, 1])
def test_fused_keys_equal_hash_then_insert(cuda, oracle, variant):
    import torch

    from paper_2101_01719_b200 import SplitBlockFilter
    from paper_2101_01719_b200.filter import hash_u64_keys
    keys = torch.arange(0, 300_000, dtype=torch.int64, device=cuda) * 7919
    a = SplitBlockFilter(4099, hasher_id=1)
    a.set_insert_variant(variant)
    a.add_keys(keys, 42)
    h = hash_u64_keys(keys, 42)
    want = oracle.build(4099, h.cpu().numpy().view(np.uint64))
    assert np.array_equal(a.blocks(), want)
    probes = torch.arange(1 << 32, (1 << 32) + 200_000, dtype=torch.int64, device=cuda)
    probes = torch.cat([keys[:5000], probes])
    want_res = oracle.find_hashes(want, hash_u64_keys(probes, 42).cpu().numpy().view(np.uint64))
    for fv in (0, 1, 3):
        a.set_find_variant(fv)
        assert np.array_equal(a.find_keys(probes, 42).cpu().numpy(), want_res)
        from oracle import bits_to_bytes
        bits = a.find_keys_bits(probes, 42).cpu().numpy().view(np.uint32)
        assert np.array_equal(bits_to_bytes(bits, probes.numel()), want_res)


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(4))
def test_fpp_sim_matches_reference(cuda, oracle, golden, idx):
    from paper_2101_01719_b200.fppsim import fpp_sim
    r = golden["fpp_sim"][idx]
    out = fpp_sim(r["ndv"], r["filter_bytes"], r["queries"], r["seed"], huge_ok=True)
    assert out["false_positives"] == r["false_positives"]
    assert oracle.image_crc(out["filter"].blocks(), hasher_id=1) == r["image_crc"]
    # acceptance.cpp:354-366 bands for the paper-table rows
    bands = {(100_000, 131_072): (0.0083, 0.0123), (1_000_000, 1_048_576): (0.0234, 0.0314),
             (100_000_000, 134_217_728): (0.00728, 0.01092)}
    lo, hi = bands.get((r["ndv"], r["filter_bytes"]), (0.0, 1.0))
    assert lo <= out["measured_fpp"] <= hi


def test_fppsim_sizing_arguments():
    """harness.cpp:33-47: exactly one of --bytes / --fpp; --fpp in (0, 1);
    --key-mode random64 | strings. All raised before any device work."""
    from paper_2101_01719_b200.fppsim import fpp_sim, resolve_buckets
    from paper_2101_01719_b200.tools import size_for
    with pytest.raises(ValueError):
        fpp_sim(10, 1 << 20, target_fpp=0.01)    # both
    with pytest.raises(ValueError):
        fpp_sim(10)                              # neither
    with pytest.raises(ValueError):
        fpp_sim(10, target_fpp=1.5)
    with pytest.raises(ValueError):
        fpp_sim(10, 1 << 20, key_mode="words")
    assert resolve_buckets(100_000, None, 0.01) == size_for(100_000, 0.01)
    assert resolve_buckets(0, None, 0.01) == 1
    assert resolve_buckets(5, 100, None) == 3


@pytest.mark.gpu
def test_device_counter_strings(cuda, oracle):
    """hash_key(std::to_string(c)) on the device (KeyMode::kByteStrings)."""
    from paper_2101_01719_b200.filter import hash_counter_strings
    for start in (0, 99_990, 2**32 - 5, 2**64 - 20):
        for seed in (0, 1, 12345):
            got = hash_counter_strings(start, 20, seed).cpu().numpy().view(np.uint64)
            want = [oracle.xxh64(str(start + i).encode(), seed) for i in range(20)]
            assert [int(x) for x in got] == want, (start, seed)


@pytest.mark.gpu
def test_fppsim_strings_and_target_fpp(cuda, oracle):
    from paper_2101_01719_b200.fppsim import NEGATIVE_COUNTER_BASE, fpp_sim
    from paper_2101_01719_b200.tools import size_for
    ndv, q, seed = 20_000, 50_000, 3
    r = fpp_sim(ndv, 65_536, q, seed, key_mode="strings")
    ins = np.array([oracle.xxh64(str(c).encode(), seed) for c in range(ndv)], np.uint64)
    probes = np.array([oracle.xxh64(str(NEGATIVE_COUNTER_BASE + i).encode(), seed) for i in range(q)], np.uint64)
    blocks = oracle.build(65_536 // 32, ins)
    assert r["false_positives"] == int(oracle.find_hashes(blocks, probes).sum())
    assert np.array_equal(r["filter"].blocks(), blocks)
    t = fpp_sim(100_000, None, 10_000, 1, target_fpp=0.01)
    assert t["filter_bytes"] == size_for(100_000, 0.01) * 32


@pytest.mark.gpu
def test_tools_bench_and_cli(cuda, oracle, capsys):
    from paper_2101_01719_b200 import tools
    from paper_2101_01719_b200.fppsim import NEGATIVE_COUNTER_BASE
    ndv, nbytes, seed = 200_000, 262_144, 7
    r = tools.run_bench(ndv, nbytes, seed, reps=3)
    ins = np.array([oracle.xxh64(c.to_bytes(8, "little"), seed) for c in range(ndv)], np.uint64)
    probes = np.array([oracle.xxh64((NEGATIVE_COUNTER_BASE + i).to_bytes(8, "little"), seed)
                       for i in range(100_000)], np.uint64)
    fp = int(oracle.find_hashes(oracle.build(nbytes // 32, ins), probes).sum())
    assert r["insert"]["measured_fpp"] == fp / 100_000 == r["lookup"]["measured_fpp"]
    assert r["lookup"]["million_ops_per_sec"] > 0 and r["insert"]["op"] == "insert"
    assert tools.main(["bench", "--ndv", "1000", "--bytes", "4096", "--reps", "3"]) == 0
    assert tools.main(["fpp-sim", "--ndv", "1000", "--bytes", "4096", "--queries", "1000"]) == 0
    out = capsys.readouterr().out
    assert out.count("insert   ndv=1000") == 1 and "measured/model fpp ratio:" in out
    assert tools.main(["bench", "--ndv", "1000", "--bytes", "4096", "--reps", "2"]) == 1


@pytest.mark.gpu
def test_fpp_mc_oracle(cuda):
    """The Monte-Carlo oracle on the GPU, checked the way the reference checks
    its own (model_test.cpp:174-207), plus one run at scale."""
    import math

    from paper_2101_01719_b200.fppsim import sbbf_fpp, sbbf_fpp_mc
    assert sbbf_fpp_mc(0.0, 64, 10_000, 1) == 0.0
    assert sbbf_fpp_mc(26.0, 256, 20_000, 77) == sbbf_fpp_mc(26.0, 256, 20_000, 77)
    for a in (20.0, 26.0):
        series = sbbf_fpp(a)
        mean = sum(sbbf_fpp_mc(a, 4096, 100_000, 1000 + r) for r in range(5)) / 5
        se = math.sqrt(series * (1.0 - series) / 100_000)
        assert abs(mean - series) <= 3.0 * se, (a, mean, series)
    a = 24.4140625                     # config 1 density
    got = sbbf_fpp_mc(a, 1 << 24, 100_000_000, 5)
    se = math.sqrt(sbbf_fpp(a) * (1 - sbbf_fpp(a)) / 1e8)
    assert abs(got - sbbf_fpp(a)) <= 4.0 * se, (got, sbbf_fpp(a))
    for bad in ((-1.0, 16, 100), (5.0, 0, 100), (5.0, 16, 0), (501.0, 16, 100)):
        with pytest.raises(ValueError):
            sbbf_fpp_mc(*bad)
