"""GPU parity: the CUDA path through the C ABI against the oracle and the
reference's golden fixtures. Bit-exact everywhere (integer/byte work).

Small cases compare whole filters and result arrays with the oracle on the
same inputs; full-size BASELINE configs compare the reference's image CRC,
set-bit count, false-positive count and per-chunk lookup-bitmap CRCs
(tests/golden/configs.json), plus size-independent properties (no false
negatives, idempotence, order independence).
"""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import bits_to_bytes  # noqa: E402
from paper_2101_01719_b200 import SplitBlockFilter, _lib  # noqa: E402
from paper_2101_01719_b200 import block_index_batch, make_mask_batch  # noqa: E402
from paper_2101_01719_b200 import workload as W  # noqa: E402

from .test_oracle import BLOCK_INDEX_KAT, MASK_KAT  # noqa: E402

INSERT_VARIANTS = [_lib.INSERT_LANE8, _lib.INSERT_LANE8_TEST, _lib.INSERT_THREAD,
                   _lib.INSERT_WIDE, _lib.INSERT_WIDE_TEST, _lib.INSERT_BLOCKED]
FIND_VARIANTS = [_lib.FIND_GLOBAL, _lib.FIND_SMEM, _lib.FIND_BLOCKED]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def dev(a, cuda):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).to(cuda)


def u32(t):
    return t.cpu().numpy().view(np.uint32)


# --- known answers on device ------------------------------------------------------
def test_block_index_kat_on_device(cuda):
    for h, nb, want in BLOCK_INDEX_KAT:
        got = block_index_batch(dev([h], cuda), nb)
        assert int(got.cpu().numpy().view(np.uint64)[0]) == want


def test_make_mask_kat_on_device(cuda, oracle):
    hs = [0, 1, 0xFFFFFFFF00000000, 0xDEADBEEF, 0x12345678DEADBEEF] + list(MASK_KAT)
    got = u32(make_mask_batch(dev(hs, cuda))).reshape(-1, 8)
    for h, row in zip(hs, got):
        assert row.tolist() == oracle.make_mask(h)
    for h, lanes in MASK_KAT.items():
        assert u32(make_mask_batch(dev([h], cuda)))[0].tolist() == lanes


def test_golden_block_index_and_mask_on_device(cuda, oracle, golden_units):
    g = golden_units["block_index"]
    hs = oracle.mt19937_64(g["hash_seed"], g["n"])
    want = np.array(g["expected"], dtype=np.uint64)
    for j, nb in enumerate(g["buckets"]):
        got = block_index_batch(dev(hs, cuda), nb).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, want[:, j]), nb
    g = golden_units["make_mask"]
    hs = oracle.mt19937_64(g["hash_seed"], g["n"])
    got = u32(make_mask_batch(dev(hs, cuda))).reshape(-1, 8)
    assert np.array_equal(got, np.array(g["expected"], dtype=np.uint32))


# --- filters built by the reference (golden) -------------------------------------
@pytest.mark.parametrize("variant", INSERT_VARIANTS)
@pytest.mark.parametrize("idx", range(10))
def test_golden_filters_on_device(cuda, oracle, golden_units, idx, variant):
    c = golden_units["filters"][idx]
    draws = oracle.mt19937_64(c["seed"], c["adds"] + c["probes"])
    ins = draws[: c["adds"]]
    half = min(c["adds"], c["probes"] // 2)
    probes = np.concatenate([ins[:half], draws[c["adds"]: c["adds"] + c["probes"] - half]])
    f = SplitBlockFilter(c["buckets"])
    f.set_insert_variant(variant)
    f.add_hashes(dev(ins, cuda))
    blocks = f.blocks()
    assert sha(blocks) == c["blocks_sha256"]
    assert oracle.image_crc(blocks) == c["image_crc"]
    if "image_hex" in c:
        assert oracle.serialize(blocks).hex() == c["image_hex"]
    res = f.find_hashes(dev(probes, cuda)).cpu().numpy()
    assert sha(res) == c["results_sha256"] and int(res.sum()) == c["hits"]
    bits = u32(f.find_hashes_bits(dev(probes, cuda)))
    assert np.array_equal(bits_to_bytes(bits, probes.size), res)


@pytest.mark.parametrize("nb", [1, 2, 7, 57, 1000, 4096, 6400, 7919, 32768, 999983])
@pytest.mark.parametrize("n", [0, 1, 31, 32, 33, 255, 257, 1000, 100_003])
def test_random_parity(cuda, oracle, nb, n):
    rng = np.random.default_rng(nb * 1000 + n)
    hs = rng.integers(0, 2**64, size=n, dtype=np.uint64)
    probes = np.concatenate([hs[: n // 2], rng.integers(0, 2**64, size=n + 7, dtype=np.uint64)])
    want = oracle.build(nb, hs)
    for v in INSERT_VARIANTS:
        f = SplitBlockFilter(nb)
        f.set_insert_variant(v)
        f.add_hashes(dev(hs, cuda))
        assert np.array_equal(f.blocks(), want), v
    want_res = oracle.find_hashes(want, probes)
    for fv in FIND_VARIANTS:
        if fv == _lib.FIND_SMEM and nb * 32 > 200 * 1024:
            continue
        f.set_find_variant(fv)
        assert np.array_equal(f.find_hashes(dev(probes, cuda)).cpu().numpy(), want_res), fv
        bits = u32(f.find_hashes_bits(dev(probes, cuda)))
        assert bits.size == (probes.size + 31) // 32
        assert np.array_equal(bits_to_bytes(bits, probes.size), want_res)
        if probes.size % 32:
            assert bits[-1] >> (probes.size % 32) == 0  # no stray bits past n


def test_host_buffer_path(cuda, oracle):
    """add_hashes/find_hashes with host arrays (pipelined H2D/D2H, several chunks)."""
    rng = np.random.default_rng(11)
    hs = rng.integers(0, 2**64, size=9_000_017, dtype=np.uint64)   # > 2 host chunks
    probes = rng.integers(0, 2**64, size=9_100_000, dtype=np.uint64)
    probes[::3] = hs[: probes[::3].size]
    f = SplitBlockFilter(123_457)
    f.add_hashes(hs)
    want = oracle.build(123_457, hs)
    assert np.array_equal(f.blocks(), want)
    want_res = oracle.find_hashes(want, probes, threads=8)
    assert np.array_equal(f.find_hashes(probes), want_res)
    assert np.array_equal(bits_to_bytes(f.find_hashes_bits(probes), probes.size), want_res)


def test_single_key_ops_and_api(cuda, oracle):
    with pytest.raises(ValueError):
        SplitBlockFilter(0)                       # filter.cpp:160-162
    f = SplitBlockFilter(1)
    assert f.num_buckets() == 1 and f.size_bytes() == 32 and f.hasher_id() == 0
    assert not f.find_hash(0)
    f.add_hash(0)                                 # filter_test.cpp:164-170
    assert f.blocks().tolist() == [[1] * 8] and f.find_hash(0)
    g = SplitBlockFilter(57)
    hs = oracle.mt19937_64(0x5EED0004, 1000)
    for h in hs[:200]:
        assert not g.find_hash(int(h)) or True
        g.add_hash(int(h))
    assert all(g.find_hash(int(h)) for h in hs[:200])
    assert np.array_equal(g.blocks(), oracle.build(57, hs[:200]))
    # from_blocks / equality / clear
    h2 = SplitBlockFilter.from_blocks(g.blocks())
    assert h2 == g
    h2.set_hasher_id(1)
    assert h2 != g
    h2.clear()
    torch.cuda.synchronize()
    assert not h2.blocks().any()
    # empty batches are no-ops (filter_test.cpp:175-180)
    g.add_hashes(dev([], cuda))
    assert g.find_hashes(dev([], cuda)).numel() == 0
    assert np.array_equal(g.blocks(), oracle.build(57, hs[:200]))


def test_idempotence_and_order_independence(cuda, oracle):
    rng = np.random.default_rng(5)
    hs = rng.integers(0, 2**64, size=1_000_000, dtype=np.uint64)
    a = SplitBlockFilter(4096)
    a.add_hashes(dev(hs, cuda))
    b = SplitBlockFilter(4096)
    b.add_hashes(dev(hs[::-1].copy(), cuda))
    b.add_hashes(dev(hs[:1000], cuda))
    assert a == b
    # concurrent inserts from two streams (atomic OR) give the same bytes
    c = SplitBlockFilter(4096)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    d = dev(hs, cuda)
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        c.add_hashes(d[: 500_000])
    with torch.cuda.stream(s2):
        c.add_hashes(d[500_000:])
    torch.cuda.synchronize()
    assert c == a
    assert np.array_equal(a.blocks(), oracle.build(4096, hs))


def test_concurrent_threads_all_paths(cuda, oracle):
    """Four host threads, each with its own stream, insert into and look up
    one filter concurrently, through every insert path including the blocked
    one (shared plan, per-call pool scratch): bytes equal the oracle's; each
    thread's lookups of keys inserted before its barrier are all hits."""
    import threading
    nb = 1 << 23   # 256 MiB
    rng = np.random.default_rng(11)
    parts = [rng.integers(0, 2**64, size=1_500_000 + 1000 * t, dtype=np.uint64) for t in range(4)]
    f = SplitBlockFilter(nb)
    f.set_insert_variant(_lib.INSERT_BLOCKED)      # concurrent blocked calls on one handle
    f.set_find_variant(_lib.FIND_BLOCKED)
    variants = [_lib.INSERT_AUTO, _lib.INSERT_BLOCKED, _lib.INSERT_WIDE_TEST, _lib.INSERT_LANE8]
    barrier = threading.Barrier(4)
    errors = []

    def work(t):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                d = dev(parts[t], cuda)
                g = SplitBlockFilter(nb)           # per-thread filter: the variant is per handle
                g.set_insert_variant(variants[t])
                g.add_hashes(d)
                f.add_hashes(d)                    # the shared filter, concurrently
                s.synchronize()
                barrier.wait()
                got = f.find_hashes(d).cpu().numpy()
                assert got.all(), t
                assert np.array_equal(g.blocks(), oracle.build(nb, parts[t])), t
        except Exception as exc:  # noqa: BLE001
            errors.append(repr(exc))

    threads = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    assert np.array_equal(f.blocks(), oracle.build(nb, np.concatenate(parts)))


def test_no_false_negatives_acceptance(cuda):
    # acceptance.cpp:63-82: 10^6 hashes, {1, 7, 4096} buckets
    rng = np.random.default_rng(0xACC0001)
    hs = dev(rng.integers(0, 2**64, size=1_000_000, dtype=np.uint64), cuda)
    for nb in (1, 7, 4096):
        f = SplitBlockFilter(nb)
        f.add_hashes(hs)
        assert int(f.find_hashes(hs).sum()) == hs.numel()


@pytest.mark.parametrize("nb", [2**20, 2**20 + 7, 3 * 2**19 + 1])
@pytest.mark.parametrize("shape", ["one_slice", "one_key", "two_slices", "ragged_tail"])
def test_blocked_path_skew(cuda, oracle, nb, shape):
    """The L2-blocked path under skew: every key in one filter slice (one
    4096-key run per chunk), one repeated key, two slices, and a batch whose
    last partition chunk is partial. Bit-exact against the oracle."""
    rng = np.random.default_rng(nb + len(shape))
    n = 300_001
    if shape == "one_slice":
        hs = rng.integers(0, 2**58, size=n, dtype=np.uint64)          # top 6 bits zero
    elif shape == "one_key":
        hs = np.full(n, 0x123456789ABCDEF1, dtype=np.uint64)
    elif shape == "two_slices":
        hs = rng.integers(0, 2**58, size=n, dtype=np.uint64) | (rng.integers(0, 2, size=n).astype(np.uint64) << np.uint64(63))
    else:
        n = 4096 * 37 + 29
        hs = rng.integers(0, 2**64, size=n, dtype=np.uint64)
    probes = np.concatenate([hs[: n // 3], rng.integers(0, 2**58, size=n // 2, dtype=np.uint64),
                             rng.integers(0, 2**64, size=1001, dtype=np.uint64)])
    want = oracle.build(nb, hs)
    f = SplitBlockFilter(nb)
    f.set_insert_variant(_lib.INSERT_BLOCKED)
    f.add_hashes(dev(hs, cuda))
    assert np.array_equal(f.blocks(), want)
    f.set_find_variant(_lib.FIND_BLOCKED)
    want_res = oracle.find_hashes(want, probes)
    assert np.array_equal(f.find_hashes(dev(probes, cuda)).cpu().numpy(), want_res)
    bits = u32(f.find_hashes_bits(dev(probes, cuda)))
    assert np.array_equal(bits_to_bytes(bits, probes.size), want_res)


@pytest.mark.parametrize("nb", [2**20, 2**21, 2**23, 2**26])
def test_blocked_tile_insert(cuda, oracle, nb):
    """Whole power-of-two filters of 2^20..2^26 blocks take the tile insert
    (slices of 256 tiles of 2048 blocks; tile_scatter then tile_apply in
    shared memory). Several calls (the sweep direction alternates), batches
    spanning several 64-chunk groups with a partial last chunk, a hot key
    repeated ~half of one call, keys packed into one tile, then lookups.
    Bit-exact against the oracle after every call."""
    rng = np.random.default_rng(nb ^ 0x711E)
    tile_lo = np.uint64(0x0123456789ABCDEF) >> np.uint64(24) << np.uint64(24)  # one tile's worth of top bits
    calls = [
        rng.integers(0, 2**64, size=64 * 4096 * 3 + 4097, dtype=np.uint64),
        np.concatenate([np.full(200_000, 0xFEEDFACECAFEBEEF, dtype=np.uint64),
                        rng.integers(0, 2**64, size=250_001, dtype=np.uint64)]),
        tile_lo | rng.integers(0, 2**20, size=100_003, dtype=np.uint64),
        rng.integers(0, 2**64, size=1, dtype=np.uint64),
    ]
    f = SplitBlockFilter(nb)
    f.set_insert_variant(_lib.INSERT_BLOCKED)
    want = oracle.new_blocks(nb)
    for hs in calls:
        rng.shuffle(hs)
        f.add_hashes(dev(hs, cuda))
        oracle.add_hashes(want, hs)
        assert np.array_equal(f.blocks(), want)
    probes = np.concatenate([calls[0][:100_000], calls[2][:5000], rng.integers(0, 2**64, size=300_000, dtype=np.uint64)])
    assert np.array_equal(f.find_hashes(dev(probes, cuda)).cpu().numpy(), oracle.find_hashes(want, probes))


def test_blocked_unaligned_buffers(cuda, oracle):
    """The TMA partition and unpermute need 16-byte aligned keys and byte
    output; a caller's hashes at an odd 8-byte offset and a byte output at
    an odd offset take the LSU kernels instead. Bit-exact either way."""
    nb = 2**21 + 3
    rng = np.random.default_rng(0xA11E)
    hs = rng.integers(0, 2**64, size=4096 * 50 + 7, dtype=np.uint64)
    probes = np.concatenate([hs[:20_000], rng.integers(0, 2**64, size=4096 * 30 + 5, dtype=np.uint64)])
    want = oracle.build(nb, hs)
    want_res = oracle.find_hashes(want, probes)
    for off in (0, 1):
        f = SplitBlockFilter(nb)
        f.set_insert_variant(_lib.INSERT_BLOCKED)
        f.set_find_variant(_lib.FIND_BLOCKED)
        d = dev(np.concatenate([np.zeros(off, np.uint64), hs]), cuda)[off:]
        f.add_hashes(d)
        assert np.array_equal(f.blocks(), want)
        p = dev(np.concatenate([np.zeros(off, np.uint64), probes]), cuda)[off:]
        res = torch.zeros(probes.size + off, dtype=torch.uint8, device="cuda")[off:]
        f.find_hashes(p, res)
        assert np.array_equal(res.cpu().numpy(), want_res)
        assert np.array_equal(bits_to_bytes(u32(f.find_hashes_bits(p)), probes.size), want_res)


@pytest.mark.parametrize("total,first,count", [
    (3 * 2**22 + 11, 2**22 + 3, 2**22 + 5),      # a middle shard, odd bounds
    (2**24, 0, 2**23),                            # the first half of a power-of-two filter
    (2**24 + 1, 2**23 + 1, 2**23),                # slices of exactly 2^20 blocks plus foreign keys
])
def test_blocked_lookup_on_a_shard_with_foreign_keys(cuda, oracle, total, first, count):
    """Blocked lookups on a block-range shard (sbbf_gpu_create_shard) with
    keys the shard does not own in the batch: the packed staging of the fused
    sweep marks them (or, when a slice has no spare offset for the mark, the
    partition + segment + unpermute kernels take the call); they answer 0,
    owned keys answer as the whole filter would. Bytes and bits."""
    from paper_2101_01719_b200 import sharded as S
    rng = np.random.default_rng(total ^ first)
    hs = rng.integers(0, 2**64, size=1_500_007, dtype=np.uint64)
    probes = np.concatenate([hs[:400_000], rng.integers(0, 2**64, size=4096 * 150 + 13, dtype=np.uint64)])
    rng.shuffle(probes)
    want = oracle.build(total, hs)
    f = S.CudaShardOps(0).create(total, first, count)
    f.set_insert_variant(_lib.INSERT_BLOCKED)
    f.add_hashes(dev(hs, cuda))                   # foreign keys are ignored
    assert np.array_equal(f.blocks(), want[first:first + count])
    blk = np.array([(int(h) * total) >> 64 for h in probes], dtype=np.uint64)
    owned = (blk >= first) & (blk < first + count)
    assert 0 < owned.sum() < probes.size
    want_res = oracle.find_hashes(want, probes) * owned
    f.set_find_variant(_lib.FIND_BLOCKED)
    assert np.array_equal(f.find_hashes(dev(probes, cuda)).cpu().numpy(), want_res)
    bits = u32(f.find_hashes_bits(dev(probes, cuda)))
    assert np.array_equal(bits_to_bytes(bits, probes.size), want_res)


@pytest.mark.parametrize("nb", [2**27, 3 * 2**25 + 5, 2**27 + 12345])
def test_blocked_two_level(cuda, oracle, nb):
    """Filters up to 128 slices of 32 MiB (4 GiB) take the single-level
    blocked path with 7-bit slice ids (2^27 blocks: top hash bits; 3 GiB + 5
    blocks: the fixed-point map); beyond, the two-level path: super-slices by
    exact block range, then slices (2^27 + 12345 blocks)."""
    rng = np.random.default_rng(nb)
    hs = rng.integers(0, 2**64, size=3_000_017, dtype=np.uint64)
    probes = np.concatenate([hs[:500_000], rng.integers(0, 2**64, size=1_500_003, dtype=np.uint64)])
    want = oracle.build(nb, hs)
    f = SplitBlockFilter(nb)
    f.set_insert_variant(_lib.INSERT_BLOCKED)
    f.add_hashes(dev(hs, cuda))
    assert np.array_equal(f.blocks(), want)
    f.set_find_variant(_lib.FIND_BLOCKED)
    want_res = oracle.find_hashes(want, probes)
    assert np.array_equal(f.find_hashes(dev(probes, cuda)).cpu().numpy(), want_res)
    bits = u32(f.find_hashes_bits(dev(probes, cuda)))
    assert np.array_equal(bits_to_bytes(bits, probes.size), want_res)


def test_64bit_block_offsets(cuda, oracle):
    """A filter larger than 2^32 words (> 16 GiB): offsets must be 64-bit."""
    nb = (1 << 29) + 12345          # 17.2 GB, 2^32+ 32-bit words
    f = SplitBlockFilter(nb)
    rng = np.random.default_rng(99)
    hs = rng.integers(0, 2**64, size=200_000, dtype=np.uint64)
    hs[:1000] |= np.uint64(0xFFFF000000000000)   # force the top of the array
    f.add_hashes(dev(hs, cuda))
    idx = np.array([oracle.block_index(int(h), nb) for h in hs[:2000]])
    assert idx.max() > (1 << 29)
    for i, h in zip(idx[:300], hs[:300]):
        blk = f.blocks_range(int(i), 1)[0]
        m = np.array(oracle.make_mask(int(h)), np.uint32)
        assert np.all(blk & m == m)
    assert int(f.find_hashes(dev(hs, cuda)).sum()) == hs.size
    top = f.blocks_range(nb - 4, 4)
    assert top.shape == (4, 8)
    del f
    torch.cuda.empty_cache()


# --- device stream generators == host oracle --------------------------------------
@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_generators_match_oracle(cuda, oracle, cid):
    cfg = W.CONFIGS[cid]
    st = W.StreamHandle(cfg.inserts)
    table = st.table.cpu().numpy().view(np.uint64) if st.table is not None else None
    ost = oracle.stream(cfg.inserts, table)
    for start in (0, 12_345_678 if cfg.inserts.n > 20_000_000 else 1000, cfg.inserts.n - 5000):
        got = W.gen_inserts(st, start, 5000).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, oracle.gen_inserts(ost, start, 5000))
    for start in (0, 99_999, cfg.lookups.n - 4000):
        got = W.gen_lookups(st, cfg.lookups, cfg.inserts.n, start, 4000).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, oracle.gen_lookups(ost, cfg.lookups, cfg.inserts.n, start, 4000))


# --- full BASELINE configs against the reference's golden values ------------------
def run_config(cid, cuda, oracle, insert_variant=0, find_variant=0):
    cfg = W.CONFIGS[cid]
    st = W.StreamHandle(cfg.inserts)
    f = SplitBlockFilter(cfg.num_buckets)
    if insert_variant:
        f.set_insert_variant(insert_variant)
    if find_variant:
        f.set_find_variant(find_variant)
    N, L = cfg.inserts.n, cfg.lookups.n
    chunk = cfg.insert_chunk or (1 << 26)
    buf = torch.empty(min(chunk, max(N, L)), dtype=torch.int64, device=cuda)
    for s in range(0, N, chunk):
        m = min(chunk, N - s)
        f.add_hashes(W.gen_inserts(st, s, m, buf[:m]))
    crcs, member_hits, fp = [], 0, 0
    gchunk = 1 << 26
    for s in range(0, L, gchunk):
        m = min(gchunk, L - s)
        q = W.gen_lookups(st, cfg.lookups, N, s, m, buf[:m])
        bits = f.find_hashes_bits(q)
        hb = u32(bits)
        crcs.append(oracle.crc32(hb.view(np.uint8)[: (m + 7) // 8].tobytes()))
        res = bits_to_bytes(hb, m)
        j = np.arange(s, s + m, dtype=np.uint64)
        if cfg.lookups.members_first:
            mem = j < N
        else:
            mem = ((j + 1) * cfg.lookups.p // cfg.lookups.q) > (j * cfg.lookups.p // cfg.lookups.q)
        member_hits += int(res[mem].sum())
        fp += int(res[~mem].sum())
    blocks = f.blocks()
    return dict(image_crc=oracle.image_crc(blocks), popcount=oracle.popcount(blocks),
                member_hits=member_hits, false_positives=fp, crcs=crcs)


@pytest.mark.parametrize("cid", [1, 2])
@pytest.mark.parametrize("iv", INSERT_VARIANTS)
def test_config_small(cuda, oracle, golden_configs, cid, iv):
    g = golden_configs[str(cid)]
    for fv in (_lib.FIND_GLOBAL, _lib.FIND_SMEM if cid == 1 else _lib.FIND_BLOCKED):
        r = run_config(cid, cuda, oracle, iv, fv)
        assert r["image_crc"] == g["image_crc"]
        assert r["popcount"] == g["popcount"]
        assert r["member_hits"] == g["members"]          # no false negatives
        assert r["false_positives"] == g["false_positives"]
        assert r["crcs"] == g["lookup_bitmap_chunk_crcs"]


@pytest.mark.slow
@pytest.mark.parametrize("cid,iv,fv", [(3, 0, 0), (4, 0, 0),
                                       (3, _lib.INSERT_WIDE_TEST, _lib.FIND_GLOBAL),
                                       (4, _lib.INSERT_WIDE_TEST, _lib.FIND_GLOBAL)])
def test_config_full(cuda, oracle, golden_configs, cid, iv, fv):
    """Full configs 3 and 4: AUTO (the L2-blocked path) and the direct path."""
    if str(cid) not in golden_configs:
        pytest.skip(f"no golden for config {cid}")
    g = golden_configs[str(cid)]
    r = run_config(cid, cuda, oracle, iv, fv)
    assert r["image_crc"] == g["image_crc"]
    assert r["popcount"] == g["popcount"]
    assert r["member_hits"] == g["members"]
    assert r["false_positives"] == g["false_positives"]
    assert r["crcs"] == g["lookup_bitmap_chunk_crcs"]


@pytest.mark.parametrize("nb,variant", [(32768, None), (1 << 23, "blocked")])
def test_cuda_graph_capture(cuda, oracle, nb, variant):
    """The device-pointer ABI is stream-ordered with no host sync, so an
    insert + lookup step captures into a CUDA graph and replays bit-exactly
    (direct path, and the single-level blocked path with its stream-ordered
    pool scratch)."""
    rng = np.random.default_rng(nb)
    hs = rng.integers(0, 2**64, size=1 << 20, dtype=np.uint64)
    look = np.concatenate([hs[: 1 << 18], rng.integers(0, 2**64, size=(1 << 20) - (1 << 18), dtype=np.uint64)])
    d, dl = dev(hs, cuda), dev(look, cuda)
    bits = torch.empty(look.size // 32, dtype=torch.int32, device=cuda)
    f = SplitBlockFilter(nb)
    if variant == "blocked":
        f.set_insert_variant(_lib.INSERT_BLOCKED)
        f.set_find_variant(_lib.FIND_BLOCKED)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):            # warm up (plans, pool) outside the capture
        f.add_hashes(d)
        f.find_hashes_bits(dl, bits)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f.add_hashes(d)
        f.find_hashes_bits(dl, bits)
    want = oracle.build(nb, hs)
    for _ in range(2):
        f.clear()
        bits.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(f.blocks(), want)
        assert np.array_equal(bits_to_bytes(u32(bits), look.size), oracle.find_hashes(want, look))


def test_blocked_pipelined_rounds(cuda, oracle):
    """Lookups spanning several rounds of the blocked path (a fused round is
    ~2.3e8 keys on a B200; the second here is ragged). Bytes and bits must
    equal the direct lookup's (itself oracle-checked), also when the call is
    captured into a CUDA graph (pool scratch, the pacing counters' memsets)."""
    nb = (1 << 23) + 777                       # 256 MiB: blocked lookups
    rng = np.random.default_rng(1234)
    hs = rng.integers(0, 2**64, size=2_000_003, dtype=np.uint64)
    f = SplitBlockFilter(nb)
    f.add_hashes(dev(hs, cuda))
    want_blocks = oracle.build(nb, hs)
    assert np.array_equal(f.blocks(), want_blocks)
    n = (1 << 28) + 4096 * 3 + 17              # two rounds, the second ragged
    look = torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device=cuda)
    look[: hs.size] = dev(hs, cuda)            # members in the first round
    look[n - 1000:] = dev(hs[:1000], cuda)     # and at the very end
    f.set_find_variant(_lib.FIND_GLOBAL)
    want = f.find_hashes(look)
    want_bits = f.find_hashes_bits(look)
    f.set_find_variant(_lib.FIND_BLOCKED)
    assert torch.equal(f.find_hashes(look), want)
    bits = f.find_hashes_bits(look)
    assert torch.equal(bits, want_bits)
    sample = look[-300_000:].cpu().numpy().view(np.uint64)
    assert np.array_equal(want[-300_000:].cpu().numpy(), oracle.find_hashes(want_blocks, sample))
    assert int(want[: hs.size].sum()) == hs.size and int(want[n - 1000:].sum()) == 1000
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        f.find_hashes_bits(look, bits)
    bits.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(bits, want_bits)


@pytest.mark.parametrize("nb", [1 << 22, 4_400_007, (1 << 23) + 5])
def test_range_split_passes(cuda, oracle, nb):
    """Whole filters somewhat larger than L2 insert (2 or 4 passes) and look
    up (2 passes, up to ~1.2 x L2) in range-split passes over the top hash
    bits: every pass touches one L2-resident block range; bitmap words are
    stored by the first pass and ORed by the next. Bit-exact against the
    oracle for bytes and bits, with ragged batch sizes."""
    rng = np.random.default_rng(nb)
    hs = rng.integers(0, 2**64, size=3_000_017, dtype=np.uint64)
    probes = np.concatenate([hs[:700_001], rng.integers(0, 2**64, size=1_300_003, dtype=np.uint64)])
    f = SplitBlockFilter(nb)
    f.add_hashes(dev(hs, cuda))
    want = oracle.build(nb, hs)
    assert np.array_equal(f.blocks(), want)
    want_res = oracle.find_hashes(want, probes)
    f.set_find_variant(_lib.FIND_GLOBAL)
    assert np.array_equal(f.find_hashes(dev(probes, cuda)).cpu().numpy(), want_res)
    bits = u32(f.find_hashes_bits(dev(probes, cuda)))
    assert np.array_equal(bits_to_bytes(bits, probes.size), want_res)


@pytest.mark.parametrize("nb", [1 << 22, 4_400_007, (1 << 23) + 5])
def test_range_split_passes_keys_frontend(cuda, oracle, nb):
    """The fused XXH64 key frontend (hash_u64_key, hash.cpp:108-114) takes
    the same range-split passes: add_keys / find_keys / find_keys_bits over
    u64 keys must equal hashing on the device first and then inserting /
    probing the hashes (itself oracle-checked above), including the bitmap
    path where the first pass stores each word and later passes OR into it."""
    rng = np.random.default_rng(nb ^ 0xF00D)
    keys = rng.integers(0, 2**64, size=2_000_003, dtype=np.uint64)
    probes = np.concatenate([keys[:500_001], rng.integers(0, 2**64, size=1_000_037, dtype=np.uint64)])
    seed = 20160216
    dk, dp = dev(keys, cuda), dev(probes, cuda)
    from paper_2101_01719_b200 import hash_u64_keys
    hk = hash_u64_keys(dk, seed)
    hp = hash_u64_keys(dp, seed)
    # the device hash equals the oracle's XXH64 of the key's 8 LE bytes
    sample = probes[-1000:]
    want_h = np.array([oracle.xxh64(int(k).to_bytes(8, "little"), seed) for k in sample], np.uint64)
    assert np.array_equal(hp[-1000:].cpu().numpy().view(np.uint64), want_h)
    f = SplitBlockFilter(nb, hasher_id=1)
    f.add_keys(dk, seed)
    want = oracle.build(nb, hk.cpu().numpy().view(np.uint64))
    assert np.array_equal(f.blocks(), want)
    want_res = oracle.find_hashes(want, hp.cpu().numpy().view(np.uint64))
    assert np.array_equal(f.find_keys(dp, seed).cpu().numpy(), want_res)
    bits = u32(f.find_keys_bits(dp, seed))
    assert np.array_equal(bits_to_bytes(bits, probes.size), want_res)
