"""Config 5 (BASELINE.json's sharded config) bit-exact against the reference.

The 8 GiB filter (2^28 blocks) takes 8e9 inserts of splitmix64(9) and 8e9
lookups (25 % members, non-members from splitmix64(10)). Golden values are
the reference's own outputs (tests/golden/make_golden.py --cfg5: image CRC
of the built filter, false positives over the 6e9 non-members, member hits,
and the CRC of every 2^26-key lookup bitmap chunk).

One B200 holds the whole filter, so config 5 runs twice here:
  * through the direct ABI (filters beyond 4 GiB take the two-level blocked
    path: super-slices, then 32 MiB slices), and
  * through ShardedFilter(fused=True) at world 1 (the multi-GPU layer's peer
    window dispatch with a single owner).
The sharded bench's per-world samples (prefixes of the same streams) are
checked by bench.py's `parity` field against golden["samples"].
"""
import json
import os
import zlib

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")

from paper_2101_01719_b200 import SplitBlockFilter  # noqa: E402
from paper_2101_01719_b200 import workload as W  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def golden5():
    with open(os.path.join(ROOT, "tests", "golden", "config5.json")) as fh:
        return json.load(fh)


def member_mask_words(start: int, nwords: int, p: int, q: int) -> np.ndarray:
    """Bitmap words of the member positions [start, start + 32*nwords) under
    the exact-fraction rule (position j is a member iff floor((j+1)p/q) >
    floor(jp/q)); for p/q = 1/4 and start % 32 == 0 every word is 0x88888888."""
    j = np.arange(start, start + 32 * nwords, dtype=np.uint64)
    mem = ((j + 1) * p // q) > (j * p // q)
    return np.packbits(mem, bitorder="little").view(np.uint32)


def sweep(insert, find_bits, image_crc, cuda, chunk=1 << 26):
    """Insert config 5's stream, then look it up chunk by chunk; returns the
    reference-comparable summary."""
    cfg = W.CONFIGS[5]
    st = W.StreamHandle(cfg.inserts)
    N, L = cfg.inserts.n, cfg.lookups.n
    buf = torch.empty(chunk, dtype=torch.int64, device=cuda)
    for s in range(0, N, chunk):
        m = min(chunk, N - s)
        insert(W.gen_inserts(st, s, m, buf[:m]))
    crc = image_crc()
    crcs, mh, fp = [], 0, 0
    mmask = None
    for s in range(0, L, chunk):
        m = min(chunk, L - s)
        q = W.gen_lookups(st, cfg.lookups, N, s, m, buf[:m])
        hb = find_bits(q).cpu().numpy().view(np.uint32)
        crcs.append(zlib.crc32(hb.view(np.uint8)[: (m + 7) // 8].tobytes()) & 0xFFFFFFFF)
        if mmask is None or mmask.size != hb.size:
            mmask = member_mask_words(s, hb.size, cfg.lookups.p, cfg.lookups.q)
        assert s % 32 == 0
        mh += int(np.bitwise_count(hb & mmask).sum())
        fp += int(np.bitwise_count(hb & ~mmask).sum())
    return dict(image_crc=crc, member_hits=mh, false_positives=fp, crcs=crcs)


def check(r, g):
    assert r["image_crc"] == g["image_crc"], f"image CRC {r['image_crc']:#x} != reference {g['image_crc']:#x}"
    assert r["member_hits"] == g["members"] == g["member_hits"]      # no false negatives
    assert r["false_positives"] == g["false_positives"]
    assert r["crcs"] == g["lookup_bitmap_chunk_crcs"]


def test_config5_direct_abi(cuda, golden5):
    g = golden5["5"]
    f = SplitBlockFilter(W.CONFIGS[5].num_buckets)
    r = sweep(f.add_hashes, f.find_hashes_bits, f.image_crc, cuda)
    check(r, g)
    del f
    torch.cuda.empty_cache()


def test_config5_sharded_world1(cuda, golden5):
    from paper_2101_01719_b200.sharded import ShardedFilter
    g = golden5["5"]
    chunk = 1 << 26
    sf = ShardedFilter(W.CONFIGS[5].num_buckets, fused=True, rank=0, world=1, max_batch=chunk)
    assert sf.route is not None, "fused routing must be active"
    r = sweep(sf.add_hashes, sf.find_hashes_bits, sf.shard.image_crc, cuda, chunk)
    check(r, g)
    del sf
    torch.cuda.empty_cache()
