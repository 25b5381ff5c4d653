"""Multi-GPU sharded SBBF: one process per GPU, filter partitioned by
contiguous block range, keys routed to their owner with an all-to-all
(the reference itself has no distributed mode).

Rank r of P owns global blocks ``[floor(r*B/P), floor((r+1)*B/P))`` and keeps
the global ``block_index`` (``mulhi(hash, B)``), so the shards concatenated in
rank order are byte-identical to the reference's single B-bucket filter.

insert: partition (``sbbf_shard_count`` + ``sbbf_shard_scatter``) ->
        counts all-to-all -> keys all-to-all (NCCL over NVLink) -> local insert
find:   same forward exchange (keeping source positions) -> local find (one
        byte per key, receive order) -> reverse all-to-all of the answers ->
        ``sbbf_scatter_u8`` back to source order (-> ``sbbf_pack_bits``).

Fused mode (the default on GPUs, ``PeerRoute`` / ``csrc/sbbf_route.cu``):
the partition's scatter writes each owner's run straight into that owner's
receive window — its GPU memory mapped here by CUDA IPC, written over
NVLink — so there is no staging array, no counts exchange and no host sync;
a 1-element NCCL all-reduce orders the phases on the stream:

insert: dispatch -> barrier -> insert_window
find:   dispatch -> barrier -> find_window -> barrier -> combine

``torch.distributed`` is the plumbing (NCCL on GPUs, gloo in the CPU tests);
the per-rank compute goes through ``ShardOps`` — ``CudaShardOps`` (the C ABI)
in the product. Tests inject a host restatement to exercise the exchange
logic on CPU with world_size 2.
"""
from __future__ import annotations

import ctypes as C
import os
import statistics
import time

import numpy as np

from . import _lib
from ._lib import check

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover
    torch = None
    dist = None


def shard_bounds(total_buckets: int, parts: int) -> list[int]:
    """bounds[r] = floor(r * B / P), r = 0..P (the shard of rank r is [bounds[r], bounds[r+1]))."""
    if parts < 1 or total_buckets < parts:
        raise ValueError("need 1 <= parts <= total_buckets")
    return [(total_buckets * r) // parts for r in range(parts + 1)]


def owner_of_block(b: int, total_buckets: int, parts: int) -> int:
    """Rank owning global block b: floor(((b+1)P - 1) / B)."""
    return ((b + 1) * parts - 1) // total_buckets


class ShardOps:
    """Per-rank compute used by ShardedFilter (device- or host-resident)."""

    def create(self, total: int, first: int, count: int):
        raise NotImplementedError

    def partition(self, keys, total: int, bounds: list[int], with_pos: bool):
        """-> (counts: list[int], routed keys grouped by owner, positions or None)."""
        raise NotImplementedError

    def insert(self, shard, keys) -> None:
        raise NotImplementedError

    def find(self, shard, keys):
        """-> one 0/1 byte per key (same device/type family as keys)."""
        raise NotImplementedError

    def scatter_back(self, answers, pos, n: int):
        raise NotImplementedError

    def pack_bits(self, answers):
        raise NotImplementedError

    def blocks(self, shard) -> np.ndarray:
        raise NotImplementedError

    def empty(self, n: int, dtype):
        raise NotImplementedError


class CudaShardOps(ShardOps):
    """The product path: sm_100a kernels behind the C ABI."""

    def __init__(self, device: int):
        self.device = device
        self.dev = torch.device("cuda", device)
        self._bounds_cache: dict = {}

    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)

    def create(self, total, first, count):
        from .filter import SplitBlockFilter
        f = SplitBlockFilter.__new__(SplitBlockFilter)
        f._h = C.c_void_p()
        check(_lib.lib().sbbf_gpu_create_shard(total, first, count, self.device, C.byref(f._h)),
              "sbbf_gpu_create_shard")
        f._device = self.device
        return f

    def _dev_bounds(self, bounds):
        key = tuple(bounds)
        if key not in self._bounds_cache:
            self._bounds_cache[key] = torch.tensor(bounds[:-1], dtype=torch.int64, device=self.dev)
        return self._bounds_cache[key]

    def partition(self, keys, total, bounds, with_pos):
        L = _lib.lib()
        parts = len(bounds) - 1
        n = keys.numel()
        db = self._dev_bounds(bounds)
        counts = torch.empty(parts, dtype=torch.int64, device=self.dev)
        s = self._stream()
        if parts <= 64:
            # one-call multisplit partition (count + scan + smem-staged scatter)
            scratch = torch.empty(parts, dtype=torch.int64, device=self.dev)
            routed = torch.empty(n, dtype=torch.int64, device=self.dev)
            pos = torch.empty(n, dtype=torch.int32, device=self.dev) if with_pos else None
            check(L.sbbf_shard_partition(C.c_void_p(keys.data_ptr()), n, total, C.c_void_p(db.data_ptr()),
                                         parts, C.c_void_p(counts.data_ptr()), C.c_void_p(scratch.data_ptr()),
                                         C.c_void_p(routed.data_ptr()),
                                         C.c_void_p(pos.data_ptr()) if with_pos else None, s),
                  "sbbf_shard_partition")
            return counts.tolist(), routed, pos
        check(L.sbbf_shard_count(C.c_void_p(keys.data_ptr()), n, total, C.c_void_p(db.data_ptr()),
                                 parts, C.c_void_p(counts.data_ptr()), s), "sbbf_shard_count")
        offsets = torch.cumsum(counts, 0) - counts
        cursor = torch.empty(parts, dtype=torch.int64, device=self.dev)
        routed = torch.empty(n, dtype=torch.int64, device=self.dev)
        pos = torch.empty(n, dtype=torch.int32, device=self.dev) if with_pos else None
        check(L.sbbf_shard_scatter(C.c_void_p(keys.data_ptr()), n, total, C.c_void_p(db.data_ptr()),
                                   parts, C.c_void_p(offsets.data_ptr()), C.c_void_p(cursor.data_ptr()),
                                   C.c_void_p(routed.data_ptr()),
                                   C.c_void_p(pos.data_ptr()) if with_pos else None, s),
              "sbbf_shard_scatter")
        return counts.tolist(), routed, pos

    def insert(self, shard, keys):
        check(_lib.lib().sbbf_gpu_insert_batch(shard.handle, C.c_void_p(keys.data_ptr()), keys.numel(),
                                               self._stream()), "sbbf_gpu_insert_batch")

    def find(self, shard, keys):
        out = torch.empty(keys.numel(), dtype=torch.uint8, device=self.dev)
        check(_lib.lib().sbbf_gpu_find_batch(shard.handle, C.c_void_p(keys.data_ptr()), keys.numel(),
                                             C.c_void_p(out.data_ptr()), self._stream()),
              "sbbf_gpu_find_batch")
        return out

    def scatter_back(self, answers, pos, n):
        out = torch.empty(n, dtype=torch.uint8, device=self.dev)
        check(_lib.lib().sbbf_scatter_u8(C.c_void_p(answers.data_ptr()), C.c_void_p(pos.data_ptr()), n,
                                         C.c_void_p(out.data_ptr()), self._stream()), "sbbf_scatter_u8")
        return out

    def pack_bits(self, answers):
        n = answers.numel()
        out = torch.empty((n + 31) // 32, dtype=torch.int32, device=self.dev)
        check(_lib.lib().sbbf_pack_bits(C.c_void_p(answers.data_ptr()), n, C.c_void_p(out.data_ptr()),
                                        self._stream()), "sbbf_pack_bits")
        return out

    def blocks(self, shard):
        return shard.blocks()

    def empty(self, n, dtype):
        return torch.empty(n, dtype=dtype, device=self.dev)


class PeerRoute:
    """This rank's receive window and its mappings of every peer's window
    (``sbbf_route_*`` in include/sbbf_gpu.h). One collective call = one
    ``dispatch`` on every rank, then the owner/source phases below."""

    def __init__(self, parts: int, rank: int, max_batch: int, device: int):
        self._h = C.c_void_p()
        self.parts, self.rank, self.device = parts, rank, device
        check(_lib.lib().sbbf_route_create(parts, rank, max_batch, device, C.byref(self._h)),
              "sbbf_route_create")
        self.max_batch = int(_lib.lib().sbbf_route_max_batch(self._h))

    def close(self):
        if self._h:
            _lib.lib().sbbf_route_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        check(_lib.lib().sbbf_route_ipc_handle(self._h, buf), "sbbf_route_ipc_handle")
        return bytes(buf)

    def open_peer(self, peer: int, handle: bytes):
        buf = (C.c_uint8 * 64).from_buffer_copy(handle)
        check(_lib.lib().sbbf_route_open_peer(self._h, peer, buf), "sbbf_route_open_peer")

    def link_local(self, peer: int, other: "PeerRoute"):
        check(_lib.lib().sbbf_route_link_local(self._h, peer, other._h), "sbbf_route_link_local")

    def ready(self) -> bool:
        return bool(_lib.lib().sbbf_route_ready(self._h))

    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream(torch.device("cuda", self.device)).cuda_stream)

    def dispatch(self, keys, total: int, d_bounds, keep_positions: bool):
        n = keys.numel()
        if n > self.max_batch:
            raise ValueError(f"batch of {n} keys exceeds max_batch={self.max_batch}; split it "
                             "identically on every rank")
        check(_lib.lib().sbbf_route_dispatch(self._h, C.c_void_p(keys.data_ptr()) if n else None, n, total,
                                             C.c_void_p(d_bounds.data_ptr()), int(keep_positions),
                                             self._stream()), "sbbf_route_dispatch")

    def insert_window(self, shard):
        check(_lib.lib().sbbf_route_insert_window(self._h, shard.handle, self._stream()),
              "sbbf_route_insert_window")

    def find_window(self, shard):
        check(_lib.lib().sbbf_route_find_window(self._h, shard.handle, self._stream()),
              "sbbf_route_find_window")

    def combine(self, out):
        check(_lib.lib().sbbf_route_combine(self._h, C.c_void_p(out.data_ptr()) if out.numel() else None,
                                            self._stream()), "sbbf_route_combine")


def _peer_access_everywhere(devices: list[int]) -> bool:
    for a in devices:
        for b in devices:
            if a != b and not torch.cuda.can_device_access_peer(a, b):
                return False
    return True


class ShardedFilter:
    """One rank's view of a P-way sharded filter of ``total_buckets`` buckets.

    fused: route keys through peer-memory windows (``PeerRoute``) instead of
    NCCL all-to-alls. None = on whenever the per-rank compute is the CUDA
    library and every rank's GPU can map every other's (always at world 1).
    max_batch: largest batch a rank passes per call in fused mode (window
    capacity); larger batches must be split identically on every rank."""

    def __init__(self, total_buckets: int, ops: ShardOps | None = None, group=None,
                 rank: int | None = None, world: int | None = None, fused: bool | None = None,
                 max_batch: int = 1 << 24):
        if total_buckets <= 0:
            raise ValueError("SplitBlockFilter needs at least one bucket")
        self.group = group
        init = dist is not None and dist.is_available() and dist.is_initialized()
        self.rank = rank if rank is not None else (dist.get_rank(group) if init else 0)
        self.world = world if world is not None else (dist.get_world_size(group) if init else 1)
        self.total = int(total_buckets)
        self.bounds = shard_bounds(self.total, self.world)
        self.first = self.bounds[self.rank]
        self.count = self.bounds[self.rank + 1] - self.first
        if ops is None:
            ops = CudaShardOps(torch.cuda.current_device())
        self.ops = ops
        self.shard = ops.create(self.total, self.first, self.count)
        self.last_exchange: dict = {}
        self.route = None
        fused_req = fused is True
        # one rank owns every block: no routing at all unless asked for
        self.direct = fused is None and self.world == 1 and isinstance(ops, CudaShardOps)
        if fused is None:
            fused = not self.direct and isinstance(ops, CudaShardOps) and self._peer_capable(init)
        if fused:
            if not isinstance(ops, CudaShardOps):
                raise ValueError("fused routing needs the CUDA shard ops")
            self._setup_route(init, max_batch, required=fused_req)

    def _peer_capable(self, init: bool) -> bool:
        if self.world == 1:
            return True
        if not init or dist.get_backend(self.group) != "nccl":
            return False
        devs = [None] * self.world
        dist.all_gather_object(devs, self.ops.device, group=self.group)
        return _peer_access_everywhere(devs)

    def _setup_route(self, init: bool, max_batch: int, required: bool = False):
        """Map every peer's window. The ranks agree collectively: if any rank
        cannot map a peer (e.g. GPUs hidden from each other), every rank falls
        back to the NCCL path (or raises, when fused routing was required)."""
        route, err = None, ""
        try:
            route = PeerRoute(self.world, self.rank, max_batch, self.ops.device)
        except Exception as exc:  # noqa: BLE001 - reported below, collectively
            err = repr(exc)
        if self.world > 1:
            handles = [None] * self.world
            dist.all_gather_object(handles, route.handle() if route is not None else None, group=self.group)
            if route is not None and None not in handles:
                try:
                    for peer, h in enumerate(handles):
                        if peer != self.rank:
                            route.open_peer(peer, h)
                except Exception as exc:  # noqa: BLE001
                    err = repr(exc)
            ok = [None] * self.world
            dist.all_gather_object(ok, err, group=self.group)
            err = next((e for e in ok if e), "")
        if err or route is None or not route.ready():
            if route is not None:
                route.close()
            if required:
                raise RuntimeError(f"fused routing unavailable: {err}")
            self.route = None
            self.route_error = err
            return
        self.route = route
        self._flag = torch.zeros(1, dtype=torch.int32, device=self.ops.dev)

    def _barrier(self):
        """Every rank's preceding kernels finish before any rank's following
        kernels start: a 1-element NCCL all-reduce (stream-ordered, no host
        sync); with a host backend (gloo), device sync + host barrier."""
        if self.world == 1:
            return
        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(self._flag, group=self.group)
        else:
            torch.cuda.synchronize(self.ops.dev)
            dist.barrier(group=self.group)

    # -- exchange ---------------------------------------------------------------
    def _exchange(self, payload, send_counts: list[int], recv_counts: list[int] | None = None):
        """all-to-all with uneven splits; returns (received, recv_counts)."""
        if not (dist is not None and dist.is_available() and dist.is_initialized()):
            assert self.world == 1
            return payload, send_counts
        if recv_counts is None:
            sc = torch.tensor(send_counts, dtype=torch.int64, device=payload.device)
            rc = torch.empty_like(sc)
            dist.all_to_all_single(rc, sc, group=self.group)
            recv_counts = rc.tolist()
        out = torch.empty(sum(recv_counts), dtype=payload.dtype, device=payload.device)
        dist.all_to_all_single(out, payload, output_split_sizes=recv_counts,
                               input_split_sizes=send_counts, group=self.group)
        return out, recv_counts

    # -- hot path -----------------------------------------------------------------
    def add_hashes(self, keys) -> None:
        """Insert this rank's batch (any keys; each is routed to its owner)."""
        if self.direct:
            self.ops.insert(self.shard, keys)
            return
        if self.route is not None:
            self.route.dispatch(keys, self.total, self.ops._dev_bounds(self.bounds), keep_positions=False)
            self._barrier()
            self.route.insert_window(self.shard)
            return
        counts, routed, _ = self.ops.partition(keys, self.total, self.bounds, with_pos=False)
        recv, rc = self._exchange(routed, counts)
        self.last_exchange = {"sent": counts, "received": rc}
        self.ops.insert(self.shard, recv)

    def find_hashes(self, keys):
        """0/1 byte per key of this rank's batch, in the batch's order."""
        n = keys.numel()
        if self.direct:
            return self.ops.find(self.shard, keys)
        if self.route is not None:
            self.route.dispatch(keys, self.total, self.ops._dev_bounds(self.bounds), keep_positions=True)
            self._barrier()
            self.route.find_window(self.shard)
            self._barrier()
            out = self.ops.empty(n, torch.uint8)
            self.route.combine(out)
            return out
        counts, routed, pos = self.ops.partition(keys, self.total, self.bounds, with_pos=True)
        recv, rc = self._exchange(routed, counts)
        answers = self.ops.find(self.shard, recv)
        back, _ = self._exchange(answers, rc, counts)
        self.last_exchange = {"sent": counts, "received": rc}
        return self.ops.scatter_back(back, pos, n)

    def find_hashes_bits(self, keys):
        return self.ops.pack_bits(self.find_hashes(keys))

    # -- inspection -----------------------------------------------------------------
    def local_blocks(self) -> np.ndarray:
        return self.ops.blocks(self.shard)

    def image_crc(self, hasher_id: int = 0) -> int:
        """FilterImage CRC (persist.cpp:72-88) of the gathered filter — the
        shards concatenated in rank order — without moving the blocks: every
        rank CRCs its shard on its GPU, the CRCs are all-gathered and combined
        in rank order behind the 17-byte header (collective; every rank
        returns the same value)."""
        L = _lib.lib()
        mine = self.shard.blocks_crc() if hasattr(self.shard, "blocks_crc") else None
        if mine is None:  # host shard ops (tests): CRC the local blocks on the host
            b = np.ascontiguousarray(self.local_blocks())
            mine = int(L.sbbf_crc32_update(0, b.ctypes.data_as(C.c_void_p), b.nbytes))
        crcs = [mine]
        if self.world > 1:
            crcs = [None] * self.world
            dist.all_gather_object(crcs, mine, group=self.group)
        hdr = (b"SBBF" + bytes([1]) + int(hasher_id).to_bytes(4, "little") +
               int(self.total).to_bytes(8, "little"))
        buf = (C.c_uint8 * len(hdr)).from_buffer_copy(hdr)
        crc = int(L.sbbf_crc32_update(0, C.cast(buf, C.c_void_p), len(hdr)))
        for r in range(self.world):
            n = (self.bounds[r + 1] - self.bounds[r]) * 32
            crc = int(L.sbbf_crc32_combine(crc, int(crcs[r]), n))
        return crc

    def gather_blocks(self, dst: int = 0):
        """Whole filter (num_buckets, 8) on rank `dst` (None elsewhere): the shards
        in rank order, which must equal the single-filter bytes."""
        mine = self.local_blocks()
        if self.world == 1:
            return mine
        t = torch.from_numpy(mine.view(np.int32).reshape(-1).copy())
        backend = dist.get_backend(self.group)
        if backend == "nccl":
            t = t.to(torch.device("cuda", torch.cuda.current_device()))
        sizes = [(self.bounds[r + 1] - self.bounds[r]) * 8 for r in range(self.world)]
        buf = [torch.empty(max(sizes), dtype=torch.int32, device=t.device) for _ in range(self.world)]
        padded = torch.zeros(max(sizes), dtype=torch.int32, device=t.device)
        padded[: t.numel()] = t
        dist.all_gather(buf, padded, group=self.group)
        if self.rank != dst:
            return None
        parts = [b[:s].cpu().numpy() for b, s in zip(buf, sizes)]
        return np.concatenate(parts).view(np.uint32).reshape(-1, 8)


# ---------------------------------------------------------------------------------
# bench.py --gpus N (torchrun): weak scaling, one rank per GPU
# ---------------------------------------------------------------------------------
def bench_main(args) -> dict | None:
    """The sharded bench. value = all ranks' keys / max-over-ranks device
    time; returns the JSON line on rank 0 (bench.py adds clocks and prints
    it), None elsewhere.

    config 5 (the default under torchrun, BASELINE's sharded config): the
    8 GiB filter (2^28 blocks) is split by block range over the P ranks;
    every step each rank originates a bounded sample of config 5's streams —
    ``--sample-keys`` inserts (positions [r*S, (r+1)*S) of splitmix64(9)) and
    as many lookups (25 % members of the sampled inserts, non-members from
    splitmix64(10)) — routed to their owners over NVLink.
    config 2: each rank originates a config-2 batch (1M inserts, 10M
    lookups) into a P x 1 MiB filter (routing overhead on L2-resident
    shards)."""
    from . import workload as W
    from ._lib import launch_count

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    # SBBF_BENCH_DEVICE / SBBF_BENCH_BACKEND: exercise this N>1 code path with
    # every rank on one GPU and a host backend (tests only; no timing claim)
    local = int(os.environ.get("SBBF_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    backend = os.environ.get("SBBF_BENCH_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    else:
        dist.init_process_group(backend, rank=rank, world_size=world)
    cfg = W.CONFIGS[args.config]
    if args.config == 5:
        N = L = int(getattr(args, "sample_keys", 1 << 27))
        total = cfg.num_buckets
        workload = (f"BASELINE config 5 sample: 8 GiB filter ({total} blocks) sharded over {world} rank(s) "
                    f"by block range; per rank per step {N:,} inserts (splitmix64(9) positions "
                    f"[r*{N}, (r+1)*{N})) + {L:,} lookups (25% members)")
    else:
        N, L = cfg.inserts.n, cfg.lookups.n
        total = cfg.num_buckets * world
        workload = (f"sharded: per rank BASELINE config {args.config} batch ({N:,} inserts + {L:,} lookups) "
                    f"into a {world}-way block-range sharded filter of {total} blocks")
    # rank r originates insert positions [rN, (r+1)N) of one world-wide stream
    spec = W.InsertSpec(seed=cfg.inserts.seed, n=N * world)
    st = W.StreamHandle(spec, local)
    ins = W.gen_inserts(st, rank * N, N, device=local)
    look = W.gen_lookups(st, cfg.lookups, N * world, rank * L, L, device=local)
    route = getattr(args, "route", "auto")
    f = ShardedFilter(total, fused=None if route == "auto" else route == "fused", max_batch=max(N, L))
    how = ("peer-memory windows over NVLink (fused dispatch, sbbf_route.cu)" if f.route is not None
           else "none (one rank owns every block)" if f.direct else "NCCL all-to-all")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_rd = torch.zeros(64 << 20, dtype=torch.int32, device=dev)

    def step(k_ins, k_look):
        f.add_hashes(k_ins)
        return f.find_hashes_bits(k_look)

    def cold():
        f.shard.clear()
        flush.zero_()
        flush_rd.sum()

    for _ in range(max(args.warmup, 3)):
        cold()
        step(ins, look)
    torch.cuda.synchronize(dev)
    times = []
    l0 = launch_count()
    for _ in range(args.steps):
        cold()
        dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        last_bits = step(ins, look)
        e1.record()
        torch.cuda.synchronize(dev)
        t = torch.tensor([e0.elapsed_time(e1)], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        times.append(float(t.item()))
    launches = launch_count() - l0
    ms = statistics.mean(times)
    sent = f.last_exchange.get("sent", [])
    # parity of the last timed step (config 5): the gathered filter's image
    # CRC (shard CRCs combined in rank order, no block movement) and the
    # false-positive / member-hit counts of the lookup bitmaps, against the
    # reference's golden for the same world-wide sample
    # (tests/golden/config5.json "samples", make_golden.py --cfg5)
    parity = None
    if args.config == 5:
        crc = f.image_crc()
        j = np.arange(rank * L, (rank + 1) * L, dtype=np.uint64)
        mem = ((j + 1) * cfg.lookups.p // cfg.lookups.q) > (j * cfg.lookups.p // cfg.lookups.q)
        mwords = torch.from_numpy(np.packbits(mem, bitorder="little").view(np.int32).copy()).to(dev)
        lut = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int64, device=dev)
        nwords = (L + 31) // 32
        hits = last_bits[:nwords]
        cnt = torch.stack([lut[(hits & mwords).view(torch.uint8).long()].sum(),
                           lut[(hits & ~mwords).view(torch.uint8).long()].sum()])
        dist.all_reduce(cnt)
        mh, fp = (int(x) for x in cnt.tolist())
        parity = {"image_crc": f"{crc:#010x}", "member_hits": mh, "false_positives": fp,
                  "members": world * int(mem.sum()), "nonmembers": world * L - world * int(mem.sum()),
                  "how": "last timed step: gathered-filter image CRC (shard CRCs combined in rank order) "
                         "and lookup-bitmap counts, vs the reference on the same world-wide sample"}
        try:
            import json as _json
            with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                                   "golden", "config5.json")) as fh:
                gs = _json.load(fh)["samples"].get(str(world))
        except Exception:
            gs = None
        if gs and gs["per_rank_keys"] == N and N == L:
            parity["reference"] = {"image_crc": f"{gs['image_crc']:#010x}", "member_hits": gs["member_hits"],
                                   "false_positives": gs["false_positives"]}
            parity["matches_reference"] = (crc == gs["image_crc"] and mh == gs["member_hits"]
                                           and fp == gs["false_positives"])

    # e2e: hashes from pinned host memory, bitmap back to the host, every step
    e2e, e2e_err = [], ""
    try:
        ins_h = ins.cpu().pin_memory()
        look_h = look.cpu().pin_memory()
        res_h = torch.empty((L + 31) // 32, dtype=torch.int32, pin_memory=True)
    except RuntimeError as exc:  # e.g. page-locked memory limits on the host
        e2e_err = repr(exc)
    flags = [None] * world
    dist.all_gather_object(flags, e2e_err)
    e2e_err = next((x for x in flags if x), "")
    for k in range(args.steps + 2 if not e2e_err else 0):
        cold()
        dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        bits = step(ins_h.to(dev, non_blocking=True), look_h.to(dev, non_blocking=True))
        res_h.copy_(bits)
        torch.cuda.synchronize(dev)
        t = torch.tensor([time.perf_counter() - t0], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if k >= 2:
            e2e.append(float(t.item()))
    line = None
    if rank == 0:
        try:
            import json
            with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")) as fh:
                peak, peak_note = float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            peak, peak_note = 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"
        e2e_s = statistics.median(e2e) if e2e else float("nan")
        fwd = 8.0 * (world - 1) / world  # bytes per key crossing NVLink (forward)
        line = {
            "metric": "SBBF insert/lookup Gkeys/s (device-timed) vs random-32B-sector roofline",
            "value": world * (N + L) / (ms * 1e-3) / 1e9, "unit": "Gkeys/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded splitmix64 hash streams, generated in HBM)",
            "config": {"workload": f"{workload}; keys routed by {how}", "config_id": args.config,
                       "parallelism": f"shard{world}", "l2": "flushed between timed steps (untimed)"},
            "e2e": {"value": world * (N + L) / e2e_s / 1e9, "unit": "Gkeys/s",
                    "h2d_bytes_per_step": 8 * (N + L), "d2h_bytes_per_step": 4 * ((L + 31) // 32),
                    "ms_per_step": e2e_s * 1e3, "note": "per rank; max over ranks of wall time",
                    **({"error": e2e_err} if e2e_err else {})},
            "roofline": {"bound": "hbm", "kernel": "whole sharded step (partition + exchange + insert + probe)",
                         "routing": how,
                         "achieved": (64.0 * N + 32.0 * L) / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": (64.0 * N + 32.0 * L) / (ms * 1e-3) / 1e9 / peak, "traffic": None,
                         "bytes_per_key": (64.0 * N + 32.0 * L) / (N + L), "peak_note": peak_note,
                         "bytes_note": ("north-star roofline per rank: one random 32-B sector per lookup, a "
                                        "32-B read-modify-write (64 B) per insert, against one GPU's HBM"),
                         "nvlink": {"bytes_per_step_per_rank": (N + L) * fwd + L * (world - 1) / world,
                                    "bytes_note": "computed, not measured: keys whose owner is another rank "
                                                  "(8 B each way out) plus their 1-B answers back",
                                    "achieved_gbs": ((N + L) * fwd + L * (world - 1) / world) / (ms * 1e-3) / 1e9,
                                    "peer_peak_gbs": 900.0}},
            "collective": {"backend": dist.get_backend(), "world": dist.get_world_size(),
                           "nccl_version": ".".join(str(x) for x in torch.cuda.nccl.version())
                           if backend == "nccl" else None},
            "gpu_launches": launches, "time": "max over ranks of CUDA-event step time",
            "parity": parity,
            "last_exchange_sent_keys": sent,
        }
    dist.destroy_process_group()
    return line
