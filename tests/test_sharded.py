"""Sharded (multi-GPU) filter: exchange logic on CPU with gloo (world_size 2
and 3), routing kernels and the NCCL self-exchange on one GPU.

The CPU tests run the real ShardedFilter (paper_2101_01719_b200/sharded.py)
with an injected host restatement of the per-rank compute (numpy), and check
the gathered shards and every lookup answer against the oracle's
single-filter result. Only the exchange/partition logic is under test there;
the GPU tests cover the CUDA routing kernels.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2101_01719_b200 import sharded as S

SEEDS = np.array([0x44974D91, 0x47B6137B, 0xA2B7289D, 0x8824AD5B,
                  0x2DF1424B, 0x705495C7, 0x5C6BFB31, 0x9EFC4947], dtype=np.uint32)


def mulhi64(a: np.ndarray, b: int) -> np.ndarray:
    """floor(a*b / 2^64) with 32-bit limbs (vectorised)."""
    a = a.astype(np.uint64)
    M = np.uint64(0xFFFFFFFF)
    al, ah = a & M, a >> np.uint64(32)
    bl, bh = np.uint64(b & 0xFFFFFFFF), np.uint64(b >> 32)
    ll, lh, hl, hh = al * bl, al * bh, ah * bl, ah * bh
    mid = (ll >> np.uint64(32)) + (lh & M) + (hl & M)
    return hh + (lh >> np.uint64(32)) + (hl >> np.uint64(32)) + (mid >> np.uint64(32))


def masks(h: np.ndarray) -> np.ndarray:
    low = (h & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    return (np.uint32(1) << ((low[:, None] * SEEDS[None, :]) >> np.uint32(27))).astype(np.uint32)


class HostShardOps(S.ShardOps):
    """Numpy restatement of the per-rank compute (test double for CudaShardOps)."""

    def create(self, total, first, count):
        return {"total": total, "first": first, "count": count,
                "blocks": np.zeros((count, 8), np.uint32)}

    def partition(self, keys, total, bounds, with_pos):
        h = keys.numpy().view(np.uint64)
        b = mulhi64(h, total)
        owner = np.searchsorted(np.array(bounds[:-1], np.uint64), b, side="right") - 1
        order = np.argsort(owner, kind="stable")
        counts = np.bincount(owner, minlength=len(bounds) - 1).tolist()
        routed = torch.from_numpy(h[order].view(np.int64).copy())
        pos = torch.from_numpy(order.astype(np.int32)) if with_pos else None
        return counts, routed, pos

    def _local(self, shard, h):
        b = mulhi64(h, shard["total"]) - np.uint64(shard["first"])
        assert np.all(b < np.uint64(shard["count"])), "a key reached the wrong shard"
        return b.astype(np.int64)

    def insert(self, shard, keys):
        h = keys.numpy().view(np.uint64)
        if h.size:
            np.bitwise_or.at(shard["blocks"], self._local(shard, h), masks(h))

    def find(self, shard, keys):
        h = keys.numpy().view(np.uint64)
        if not h.size:
            return torch.zeros(0, dtype=torch.uint8)
        blk = shard["blocks"][self._local(shard, h)]
        m = masks(h)
        return torch.from_numpy(np.all((blk & m) == m, axis=1).astype(np.uint8))

    def scatter_back(self, answers, pos, n):
        out = np.zeros(n, np.uint8)
        out[pos.numpy()] = answers.numpy()
        return torch.from_numpy(out)

    def pack_bits(self, answers):
        a = answers.numpy()
        return torch.from_numpy(np.packbits(a, bitorder="little").view(np.uint8))

    def blocks(self, shard):
        return shard["blocks"]


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, n_ins, n_look, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(1000 + rank)
        ins = rng.integers(0, 2**64, size=n_ins, dtype=np.uint64)
        f = S.ShardedFilter(total, ops=HostShardOps())
        f.add_hashes(torch.from_numpy(ins.view(np.int64)))
        dist.barrier()
        look = np.concatenate([ins[: n_look // 2], rng.integers(0, 2**64, size=n_look - n_look // 2,
                                                                  dtype=np.uint64)])
        ans = f.find_hashes(torch.from_numpy(look.view(np.int64))).numpy()
        full = f.gather_blocks(0)
        crc = f.image_crc()   # collective: shard CRCs combined in rank order
        q.put((rank, ins, look, ans, full, f.first, f.count, f.last_exchange, crc))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,total", [(2, 4096), (2, 1001), (3, 7919)])
def test_gloo_sharded_matches_oracle(oracle, world, total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, 20_000, 10_000, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort(key=lambda x: x[0])
    all_ins = np.concatenate([g[1] for g in got])
    want = oracle.build(total, all_ins)
    full = got[0][4]
    assert full.shape == (total, 8)
    assert np.array_equal(full, want)                     # shards concatenate to the reference filter
    assert oracle.image_crc(full) == oracle.image_crc(want)
    # the gathered image CRC without moving blocks, identical on every rank
    assert all(g[8] == oracle.image_crc(want) for g in got)
    for rank, ins, look, ans, *_ in got:
        assert np.array_equal(ans, oracle.find_hashes(want, look)), rank
        assert ans[: len(look) // 2].all()               # no false negatives across ranks
    bounds = S.shard_bounds(total, world)
    for rank, *_rest in got:
        first, count = got[rank][5], got[rank][6]
        assert (first, count) == (bounds[rank], bounds[rank + 1] - bounds[rank])
    # exchange bookkeeping: what rank a sent to b is what b received from a
    for a in range(world):
        for b in range(world):
            assert got[a][7]["sent"][b] == got[b][7]["received"][a]


def test_bounds_and_owner():
    for total in (1, 7, 4096, 1001, 2**28, 2**28 + 3):
        for parts in (1, 2, 3, 4, 8):
            if parts > total:
                continue
            b = S.shard_bounds(total, parts)
            assert b[0] == 0 and b[-1] == total and all(x <= y for x, y in zip(b, b[1:]))
            for blk in {0, total - 1, total // 2, total // 3, max(0, b[min(1, parts)] - 1)}:
                r = S.owner_of_block(blk, total, parts)
                assert b[r] <= blk < b[r + 1]


# ---------------------------------------------------------------------------------
# GPU: routing kernels, multi-shard on one device, NCCL self-exchange
# ---------------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_cuda_partition_kernels(cuda, parts):
    ops = S.CudaShardOps(0)
    total = 2**20 + 17
    rng = np.random.default_rng(parts)
    h = rng.integers(0, 2**64, size=1_000_003, dtype=np.uint64)
    d = torch.from_numpy(h.view(np.int64)).to(cuda)
    bounds = S.shard_bounds(total, parts)
    counts, routed, pos = ops.partition(d, total, bounds, with_pos=True)
    host = HostShardOps()
    want_counts, _, _ = host.partition(torch.from_numpy(h.view(np.int64)), total, bounds, True)
    assert counts == want_counts
    r = routed.cpu().numpy().view(np.uint64)
    p = pos.cpu().numpy().astype(np.int64)
    assert np.array_equal(np.sort(p), np.arange(h.size))         # a permutation
    assert np.array_equal(r, h[p])                               # routed[i] = h[pos[i]]
    off = np.concatenate([[0], np.cumsum(counts)])
    blk = mulhi64(r, total)
    for k in range(parts):
        seg = blk[off[k]:off[k + 1]]
        assert np.all(seg >= bounds[k]) and np.all(seg < bounds[k + 1])


@pytest.mark.gpu
@pytest.mark.parametrize("parts", [2, 4, 8])
def test_multi_shard_one_gpu(cuda, oracle, parts):
    """P shards on one GPU fed by the routing kernels (no collective): the
    concatenated shards equal the single filter; lookups agree."""
    ops = S.CudaShardOps(0)
    total = 32768 * parts
    rng = np.random.default_rng(77)
    h = rng.integers(0, 2**64, size=2_000_000, dtype=np.uint64)
    look = np.concatenate([h[:500_000], rng.integers(0, 2**64, size=500_000, dtype=np.uint64)])
    bounds = S.shard_bounds(total, parts)
    shards = [ops.create(total, bounds[r], bounds[r + 1] - bounds[r]) for r in range(parts)]
    counts, routed, _ = ops.partition(torch.from_numpy(h.view(np.int64)).to(cuda), total, bounds, False)
    off = np.concatenate([[0], np.cumsum(counts)])
    for r in range(parts):
        ops.insert(shards[r], routed[off[r]:off[r + 1]])
    full = np.concatenate([s.blocks() for s in shards])
    want = oracle.build(total, h)
    assert np.array_equal(full, want)
    dl = torch.from_numpy(look.view(np.int64)).to(cuda)
    counts, routed, pos = ops.partition(dl, total, bounds, True)
    off = np.concatenate([[0], np.cumsum(counts)])
    answers = torch.cat([ops.find(shards[r], routed[off[r]:off[r + 1]]) for r in range(parts)])
    back = ops.scatter_back(answers, pos, look.size).cpu().numpy()
    assert np.array_equal(back, oracle.find_hashes(want, look))
    bits = ops.pack_bits(ops.scatter_back(answers, pos, look.size)).cpu().numpy().view(np.uint32)
    from oracle import bits_to_bytes
    assert np.array_equal(bits_to_bytes(bits, look.size), back)
    # keys a shard does not own: ignored by insert, answer 0 in find
    before = shards[0].blocks()
    ops.insert(shards[0], routed[off[-2]:off[-1]])
    assert np.array_equal(shards[0].blocks(), before)
    assert int(ops.find(shards[0], routed[off[-2]:off[-1]]).sum()) == 0


@pytest.mark.gpu
def test_nccl_self_exchange(cuda, oracle):
    """The full ShardedFilter path over NCCL at world_size 1 (self-exchange)."""
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    try:
        rng = np.random.default_rng(5)
        h = rng.integers(0, 2**64, size=1_000_000, dtype=np.uint64)
        f = S.ShardedFilter(32768, fused=False)
        assert f.route is None
        f.add_hashes(torch.from_numpy(h.view(np.int64)).to(cuda))
        want = oracle.build(32768, h)
        assert np.array_equal(f.gather_blocks(), want)
        look = np.concatenate([h[:1000], rng.integers(0, 2**64, size=100_000, dtype=np.uint64)])
        ans = f.find_hashes(torch.from_numpy(look.view(np.int64)).to(cuda)).cpu().numpy()
        assert np.array_equal(ans, oracle.find_hashes(want, look))
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------------
# GPU: fused dispatch over peer-memory windows (csrc/sbbf_route.cu)
# ---------------------------------------------------------------------------------
def _linked_routes(parts, max_batch):
    routes = [S.PeerRoute(parts, r, max_batch, 0) for r in range(parts)]
    for r in range(parts):
        for q in range(parts):
            routes[r].link_local(q, routes[q])
        assert routes[r].ready()
    return routes


@pytest.mark.gpu
@pytest.mark.parametrize("parts,total", [(1, 32768), (2, 65536), (3, 7919 * 3), (8, 2**18 + 5)])
def test_fused_route_multi_shard_one_gpu(cuda, oracle, parts, total):
    """P ranks simulated by P route contexts + shards in one process: every
    source's scatter writes into every owner's window; the concatenated
    shards equal the single filter and every source gets the oracle's
    answers. Ragged batches (one source empty), two calls of each kind so
    both window parities are used."""
    ops = S.CudaShardOps(0)
    bounds = S.shard_bounds(total, parts)
    db = ops._dev_bounds(bounds)
    shards = [ops.create(total, bounds[r], bounds[r + 1] - bounds[r]) for r in range(parts)]
    routes = _linked_routes(parts, 300_000)
    rng = np.random.default_rng(parts * 31 + 1)
    sizes = [0 if (parts > 1 and r == 1) else int(rng.integers(1, 250_000)) for r in range(parts)]
    all_ins = []
    for call in range(2):
        batch = [rng.integers(0, 2**64, size=n, dtype=np.uint64) for n in sizes]
        all_ins += batch
        dev = [torch.from_numpy(b.view(np.int64)).to(cuda) for b in batch]
        for r in range(parts):
            routes[r].dispatch(dev[r], total, db, keep_positions=False)
        for r in range(parts):
            routes[r].insert_window(shards[r])
        torch.cuda.synchronize()
        want = oracle.build(total, np.concatenate(all_ins))
        full = np.concatenate([s.blocks() for s in shards])
        assert np.array_equal(full, want), f"call {call}"
    hits = np.concatenate(all_ins)
    for call in range(2):
        looks = []
        for r in range(parts):
            m = int(rng.integers(0, 200_000)) if r != 0 else 1
            half = min(m // 2, hits.size)
            looks.append(np.concatenate([hits[rng.integers(0, hits.size, size=half)],
                                         rng.integers(0, 2**64, size=m - half, dtype=np.uint64)]))
        dev = [torch.from_numpy(x.view(np.int64)).to(cuda) for x in looks]
        for r in range(parts):
            routes[r].dispatch(dev[r], total, db, keep_positions=True)
        for r in range(parts):
            routes[r].find_window(shards[r])
        outs = [torch.empty(x.size, dtype=torch.uint8, device=cuda) for x in looks]
        for r in range(parts):
            routes[r].combine(outs[r])
        for r in range(parts):
            assert np.array_equal(outs[r].cpu().numpy(), oracle.find_hashes(want, looks[r])), (call, r)
    for rt in routes:
        rt.close()


@pytest.mark.gpu
def test_fused_route_errors(cuda):
    from paper_2101_01719_b200._lib import SbbfError
    a = S.PeerRoute(2, 0, 1000, 0)
    b = S.PeerRoute(2, 1, 5000, 0)
    assert a.max_batch == 1024                      # rounded up to a multiple of 256
    ops = S.CudaShardOps(0)
    db = ops._dev_bounds(S.shard_bounds(4096, 2))
    keys = torch.zeros(10, dtype=torch.int64, device=cuda)
    with pytest.raises(SbbfError):                  # peer 1 not linked yet
        a.dispatch(keys, 4096, db, False)
    with pytest.raises(SbbfError):                  # capacities differ
        a.link_local(1, b)
    with pytest.raises(SbbfError):                  # bad geometry
        S.PeerRoute(2, 2, 1000, 0)
    with pytest.raises(ValueError):                 # over max_batch
        a.dispatch(torch.zeros(2000, dtype=torch.int64, device=cuda), 4096, db, False)
    with pytest.raises(SbbfError):                  # combine needs a lookup dispatch
        a.combine(torch.empty(1, dtype=torch.uint8, device=cuda))
    a.close()
    b.close()


@pytest.mark.gpu
def test_fused_sharded_filter_world1(cuda, oracle):
    """ShardedFilter picks the fused route by default; with and without an
    NCCL process group it matches the oracle."""
    rng = np.random.default_rng(9)
    h = rng.integers(0, 2**64, size=700_000, dtype=np.uint64)
    look = np.concatenate([h[:5000], rng.integers(0, 2**64, size=300_000, dtype=np.uint64)])
    want = oracle.build(32768, h)
    d = S.ShardedFilter(32768)                      # world 1 default: no routing at all
    assert d.direct and d.route is None
    d.add_hashes(torch.from_numpy(h.view(np.int64)).to(cuda))
    assert np.array_equal(d.gather_blocks(), want)
    assert np.array_equal(d.find_hashes(torch.from_numpy(look.view(np.int64)).to(cuda)).cpu().numpy(),
                          oracle.find_hashes(want, look))
    f = S.ShardedFilter(32768, fused=True)
    assert f.route is not None
    f.add_hashes(torch.from_numpy(h.view(np.int64)).to(cuda))
    assert np.array_equal(f.gather_blocks(), want)
    ans = f.find_hashes(torch.from_numpy(look.view(np.int64)).to(cuda)).cpu().numpy()
    assert np.array_equal(ans, oracle.find_hashes(want, look))
    bits = f.find_hashes_bits(torch.from_numpy(look.view(np.int64)).to(cuda)).cpu().numpy().view(np.uint32)
    from oracle import bits_to_bytes
    assert np.array_equal(bits_to_bytes(bits, look.size), ans)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    try:
        g = S.ShardedFilter(32768, fused=True)
        assert g.route is not None
        g.add_hashes(torch.from_numpy(h.view(np.int64)).to(cuda))
        assert np.array_equal(g.gather_blocks(), want)
        ans = g.find_hashes(torch.from_numpy(look.view(np.int64)).to(cuda)).cpu().numpy()
        assert np.array_equal(ans, oracle.find_hashes(want, look))
        n = S.ShardedFilter(32768, fused=False)     # the NCCL all-to-all path still works
        n.add_hashes(torch.from_numpy(h.view(np.int64)).to(cuda))
        assert np.array_equal(n.gather_blocks(), want)
    finally:
        dist.destroy_process_group()


def _ipc_worker(rank, world, port, total, q):
    """One process per rank on the same GPU: windows mapped across processes
    with CUDA IPC handles (the multi-GPU plumbing), phases ordered by host
    barriers (gloo); no kernel ever waits on another process."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        rng = np.random.default_rng(500 + rank)
        ins = rng.integers(0, 2**64, size=150_000 + 1000 * rank, dtype=np.uint64)
        f = S.ShardedFilter(total, fused=True, max_batch=1 << 18)
        assert f.route is not None and f.route.ready()
        f.add_hashes(torch.from_numpy(ins.view(np.int64)).to(dev))
        look = np.concatenate([ins[:20_000], rng.integers(0, 2**64, size=60_000, dtype=np.uint64)])
        ans = f.find_hashes(torch.from_numpy(look.view(np.int64)).to(dev)).cpu().numpy()
        q.put((rank, ins, look, ans, f.local_blocks(), f.first))
        dist.barrier()
        f.route.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,total", [(2, 65536), (3, 7919 * 3)])
def test_fused_ipc_processes(cuda, oracle, world, total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got.sort(key=lambda x: x[0])
    want = oracle.build(total, np.concatenate([g[1] for g in got]))
    full = np.concatenate([g[4] for g in got])
    assert np.array_equal(full, want)
    for rank, ins, look, ans, *_ in got:
        assert np.array_equal(ans, oracle.find_hashes(want, look)), rank


@pytest.mark.gpu
@pytest.mark.parametrize("forced", [False, True])
@pytest.mark.parametrize("per_source", [1_500_000, 5_300_000])
def test_fused_route_big_shards(cuda, oracle, per_source, forced):
    """Shards beyond 2 x L2 (the config-5 regime). With few keys per owner
    the window goes through the direct path (gathered); with at least half a
    key per block, the blocked path takes the source regions as they are (one
    filter sweep, no staging copy). Under AUTO these batches (below one key
    per block) keep the segment + unpermute kernels; `forced` sets the shards
    to FIND_BLOCKED, which sends the regions through the fused lookup sweep
    (packed slots with the foreign-key mark, partial chunks inside the chunk
    layout). Bit-exact either way."""
    parts, total = 2, 2 * (300 << 20) // 32 + 3
    ops = S.CudaShardOps(0)
    bounds = S.shard_bounds(total, parts)
    db = ops._dev_bounds(bounds)
    shards = [ops.create(total, bounds[r], bounds[r + 1] - bounds[r]) for r in range(parts)]
    assert all(s.size_bytes() > 2 * (126 << 20) for s in shards)
    if forced:
        from paper_2101_01719_b200 import _lib
        for s in shards:
            s.set_find_variant(_lib.FIND_BLOCKED)
    routes = _linked_routes(parts, 1 << 23)
    rng = np.random.default_rng(4242)
    batch = [rng.integers(0, 2**64, size=per_source + 77 * r, dtype=np.uint64) for r in range(parts)]
    for r in range(parts):
        routes[r].dispatch(torch.from_numpy(batch[r].view(np.int64)).to(cuda), total, db, keep_positions=False)
    for r in range(parts):
        routes[r].insert_window(shards[r])
    want = oracle.build(total, np.concatenate(batch))
    for r in range(parts):
        assert np.array_equal(shards[r].blocks(), want[bounds[r]:bounds[r + 1]]), r
    looks = [np.concatenate([batch[1 - r][:per_source // 4], rng.integers(0, 2**64, size=per_source, dtype=np.uint64)])
             for r in range(parts)]
    for r in range(parts):
        routes[r].dispatch(torch.from_numpy(looks[r].view(np.int64)).to(cuda), total, db, keep_positions=True)
    for r in range(parts):
        routes[r].find_window(shards[r])
    for r in range(parts):
        out = torch.empty(looks[r].size, dtype=torch.uint8, device=cuda)
        routes[r].combine(out)
        assert np.array_equal(out.cpu().numpy(), oracle.find_hashes(want, looks[r])), r
    for rt in routes:
        rt.close()


@pytest.mark.gpu
@pytest.mark.parametrize("total", [32768, 7919 * 5])
def test_dist_c_abi_world1(cuda, oracle, total):
    """The C++ sharded layer (sbbf_dist_*, csrc/sbbf_dist.cu) over a 1-rank
    NCCL communicator it builds itself: insert / find / find_bits / gather
    against the oracle."""
    import ctypes as C

    from oracle import bits_to_bytes
    from paper_2101_01719_b200 import _lib
    L = _lib.lib()
    uid = (C.c_uint8 * 128)()
    _lib.check(L.sbbf_dist_unique_id(uid), "unique_id")
    comm = C.c_void_p()
    _lib.check(L.sbbf_dist_comm_init(uid, 1, 0, 0, C.byref(comm)), "comm_init")
    d = C.c_void_p()
    _lib.check(L.sbbf_dist_create(comm, total, 1 << 20, 0, C.byref(d)), "dist_create")
    try:
        assert L.sbbf_dist_rank(d) == 0 and L.sbbf_dist_world(d) == 1
        rng = np.random.default_rng(total)
        h = rng.integers(0, 2**64, size=600_000, dtype=np.uint64)
        look = np.concatenate([h[:3000], rng.integers(0, 2**64, size=200_001, dtype=np.uint64)])
        dh = torch.from_numpy(h.view(np.int64)).to(cuda)
        dl = torch.from_numpy(look.view(np.int64)).to(cuda)
        s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(L.sbbf_dist_insert(d, C.c_void_p(dh.data_ptr()), h.size, s), "dist_insert")
        out = torch.empty(look.size, dtype=torch.uint8, device=cuda)
        _lib.check(L.sbbf_dist_find(d, C.c_void_p(dl.data_ptr()), look.size, C.c_void_p(out.data_ptr()), s),
                   "dist_find")
        bits = torch.empty((look.size + 31) // 32, dtype=torch.int32, device=cuda)
        _lib.check(L.sbbf_dist_find_bits(d, C.c_void_p(dl.data_ptr()), look.size, C.c_void_p(bits.data_ptr()), s),
                   "dist_find_bits")
        torch.cuda.synchronize()
        want = oracle.build(total, h)
        full = np.zeros((total, 8), np.uint32)
        _lib.check(L.sbbf_dist_gather(d, full.ctypes.data_as(C.c_void_p), 0), "dist_gather")
        assert np.array_equal(full, want)
        want_res = oracle.find_hashes(want, look)
        assert np.array_equal(out.cpu().numpy(), want_res)
        assert np.array_equal(bits_to_bytes(bits.cpu().numpy().view(np.uint32), look.size), want_res)
        with pytest.raises(_lib.SbbfError):     # over max_batch
            _lib.check(L.sbbf_dist_insert(d, C.c_void_p(dh.data_ptr()), 2 << 20, s), "dist_insert")
    finally:
        L.sbbf_dist_destroy(d)
        L.sbbf_dist_comm_destroy(comm)


@pytest.mark.gpu
def test_bench_world2_code_path(cuda):
    """bench.py's torchrun (N > 1) path end to end — both ranks on this one
    GPU, a host backend for the collectives, fused IPC routing — so the
    multi-GPU line assembles; no timing claim is made from it."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SBBF_BENCH_DEVICE="0", SBBF_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
                          os.path.join(root, "bench.py"), "--gpus", "2", "--route", "fused",
                          "--sample-keys", str(1 << 20), "--steps", "2", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1                         # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["config_id"] == 5 and d["value"] > 0
    assert "peer-memory windows" in d["config"]["routing"]
    assert d["parity"]["how"] and d["parity"]["members"] > 0      # parity of the sampled step is reported


def _dist_hooks_worker(rank, world, port, total, q):
    """One rank of the C sharded layer (sbbf_dist_*) at world > 1 on ONE GPU:
    NCCL refuses two ranks on one device, so the collectives come from the
    caller (sbbf_dist_create_hooks) — a gloo process group here — while the
    data path is the product's: CUDA IPC receive windows, fused dispatch,
    owner-side window insert / find, combine."""
    import ctypes as C
    import datetime
    import traceback
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=120))
    try:
        _dist_hooks_body(rank, world, total, q)
    except BaseException:  # report instead of leaving the parent waiting
        q.put((rank, "error", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _dist_hooks_body(rank, world, total, q):
    if True:
        import ctypes as C
        from paper_2101_01719_b200 import _lib
        L = _lib.lib()
        torch.cuda.set_device(0)

        AG = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)
        BAR = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p)
        calls = {"barrier": 0, "allgather": 0}

        hook_errors = []

        def allgather(ctx, send, recv, nbytes):
            try:
                mine = torch.from_numpy(np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)), (nbytes,)).copy())
                outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(outs, mine)
                joined = torch.cat(outs).numpy()   # keep it alive across the copy
                C.memmove(recv, joined.ctypes.data, nbytes * world)
                calls["allgather"] += 1
                return 0
            except BaseException as exc:  # noqa: BLE001 - surfaced through the return code
                hook_errors.append(repr(exc))
                return 1

        def barrier(ctx, stream):
            try:
                torch.cuda.synchronize()        # this rank's queued work is done ...
                dist.barrier()                  # ... and every other rank's too
                calls["barrier"] += 1
                return 0
            except BaseException as exc:  # noqa: BLE001
                hook_errors.append(repr(exc))
                return 1

        class Hooks(C.Structure):
            _fields_ = [("rank", C.c_int), ("world", C.c_int), ("ctx", C.c_void_p), ("allgather", AG),
                        ("barrier", BAR)]

        ag, br = AG(allgather), BAR(barrier)
        hooks = Hooks(rank, world, None, ag, br)
        d = C.c_void_p()
        rc = L.sbbf_dist_create_hooks(C.byref(hooks), total, 1 << 20, 0, C.byref(d))
        assert rc == 0, (rc, L.sbbf_gpu_last_error(), hook_errors)
        assert L.sbbf_dist_rank(d) == rank and L.sbbf_dist_world(d) == world
        rng = np.random.default_rng(77 + rank)
        h = rng.integers(0, 2**64, size=300_000 + 1001 * rank, dtype=np.uint64)
        look = np.concatenate([h[:2000], rng.integers(0, 2**64, size=100_003, dtype=np.uint64)])
        dh = torch.from_numpy(h.view(np.int64)).cuda()
        dl = torch.from_numpy(look.view(np.int64)).cuda()
        s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(L.sbbf_dist_insert(d, C.c_void_p(dh.data_ptr()), h.size, s), "dist_insert")
        out = torch.empty(look.size, dtype=torch.uint8, device="cuda")
        _lib.check(L.sbbf_dist_find(d, C.c_void_p(dl.data_ptr()), look.size, C.c_void_p(out.data_ptr()), s),
                   "dist_find")
        bits = torch.empty((look.size + 31) // 32, dtype=torch.int32, device="cuda")
        _lib.check(L.sbbf_dist_find_bits(d, C.c_void_p(dl.data_ptr()), look.size, C.c_void_p(bits.data_ptr()), s),
                   "dist_find_bits")
        _lib.check(L.sbbf_dist_sync(d, s, 60_000), "dist_sync")
        crc = C.c_uint32(0)
        _lib.check(L.sbbf_dist_image_crc(d, C.byref(crc)), "dist_image_crc")
        full = np.zeros((total, 8), np.uint32) if rank == 0 else np.zeros(1, np.uint32)
        _lib.check(L.sbbf_dist_gather(d, full.ctypes.data_as(C.c_void_p), 0), "dist_gather")
        q.put((rank, h, look, out.cpu().numpy(), bits.cpu().numpy().view(np.uint32), full if rank == 0 else None,
               int(crc.value), dict(calls)))
        L.sbbf_dist_destroy(d)


@pytest.mark.gpu
@pytest.mark.parametrize("world,total", [(2, 1 << 20), (3, 7919 * 13)])
def test_dist_c_abi_world_gt1_one_gpu(cuda, oracle, world, total):
    """sbbf_dist_* at world 2 and 3 (every rank on this one GPU, collectives
    by hook): inserts routed to their owner shards through the peer windows,
    lookups answered and combined in source order, the gathered filter and
    its image CRC equal to the single-filter reference."""
    from oracle import bits_to_bytes
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_dist_hooks_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    errors = [g[2] for g in got if isinstance(g[1], str)]
    assert not errors, "\n".join(errors)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = oracle.build(total, np.concatenate([g[1] for g in got]))
    assert np.array_equal(got[0][5], want)
    assert all(g[6] == oracle.image_crc(want) for g in got)
    for rank, h, look, out, bits, _, _, calls in got:
        res = oracle.find_hashes(want, look)
        assert np.array_equal(out, res), rank
        assert np.array_equal(bits_to_bytes(bits, look.size), res), rank
        assert calls["barrier"] >= 5 and calls["allgather"] >= 2
