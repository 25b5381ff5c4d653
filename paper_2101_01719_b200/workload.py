"""BASELINE.json's five configs as seeded synthetic hash streams, generated in HBM.

Stream definitions (the builder-defined choices are listed in
DESIGN.md §5): output i of ``splitmix64(seed)`` is
``fmix(seed + (i+1)*0x9e3779b97f4a7c15)``. Inserts consume an insert stream
in order; lookups mix members (insert-stream values at uniformly chosen
positions) and non-members (a fresh seed, consumed in order) by an exact
fraction. Config 4 adds Zipf(1.1) duplicates over its first 10M keys.

Generation runs on the GPU (``sbbf_gen_inserts`` / ``sbbf_gen_lookups``);
``oracle/`` restates every stream on the host and tests compare prefixes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import InsertStream, check

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


@dataclass(frozen=True)
class InsertSpec:
    seed: int
    n: int
    fresh_prefix: int = 0
    dup_num: int = 0
    dup_den: int = 1
    dup_sel_seed: int = 0
    zipf_s: float = 0.0
    zipf_n: int = 0


@dataclass(frozen=True)
class LookupSpec:
    n: int
    nonmember_seed: int
    sel_seed: int
    p: int
    q: int
    members_first: bool = False  # config 1: all members in insert order, then non-members


@dataclass(frozen=True)
class Config:
    cid: int
    name: str
    num_buckets: int
    inserts: InsertSpec
    lookups: LookupSpec
    insert_chunk: int = 0  # 0 = one batch
    notes: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def filter_bytes(self) -> int:
        return self.num_buckets * 32


CONFIGS = {
    1: Config(1, "cfg1-100k-128KiB", 4096, InsertSpec(seed=1, n=100_000),
              LookupSpec(n=1_100_000, nonmember_seed=2, sel_seed=0, p=0, q=1, members_first=True),
              notes="100k members in insert order, then 1M non-members (seed 2)"),
    2: Config(2, "cfg2-1M-1MiB", 32_768, InsertSpec(seed=3, n=1_000_000),
              LookupSpec(n=10_000_000, nonmember_seed=4, sel_seed=104, p=1, q=2)),
    3: Config(3, "cfg3-100M-128MiB", 1 << 22, InsertSpec(seed=5, n=100_000_000),
              LookupSpec(n=1_000_000_000, nonmember_seed=6, sel_seed=106, p=1, q=10)),
    4: Config(4, "cfg4-1G-zipf-1GiB", 1 << 25,
              InsertSpec(seed=7, n=1_000_000_000, fresh_prefix=10_000_000, dup_num=20, dup_den=99,
                         dup_sel_seed=107, zipf_s=1.1, zipf_n=10_000_000),
              LookupSpec(n=2_000_000_000, nonmember_seed=8, sel_seed=108, p=1, q=2),
              insert_chunk=1 << 26,
              notes="non-member seed 8 (unused slot) is a builder choice; chunks of 2^26 keys"),
    5: Config(5, "cfg5-8G-sharded-8GiB", 1 << 28, InsertSpec(seed=9, n=8_000_000_000),
              LookupSpec(n=8_000_000_000, nonmember_seed=10, sel_seed=110, p=1, q=4),
              notes="sharded by contiguous block range across ranks"),
}


def zipf_cdf_table(s: float, n: int) -> np.ndarray:
    """Integer inverse-CDF thresholds for Zipf(s) over ranks 0..n-1:
    T[r] = floor(CDF(r) * 2^64) (last entry saturated), so rank = first r with
    u < T[r] for a uniform u64. Built once on the host in float64."""
    w = np.arange(1, n + 1, dtype=np.float64) ** (-s)
    c = np.cumsum(w)
    cdf = c / c[-1]
    t = np.empty(n, np.uint64)
    scaled = cdf * 18446744073709551616.0
    ok = scaled < 18446744073709551616.0
    t[ok] = scaled[ok].astype(np.uint64)
    t[~ok] = np.uint64(0xFFFFFFFFFFFFFFFF)
    t[-1] = np.uint64(0xFFFFFFFFFFFFFFFF)
    return t


class StreamHandle:
    """Keeps the device Zipf table alive for an InsertStream struct."""

    def __init__(self, spec: InsertSpec, device: int = 0):
        self.spec = spec
        self.table = None
        zipf_ptr = None
        if spec.dup_num:
            host = zipf_cdf_table(spec.zipf_s, spec.zipf_n)
            self.table = torch.from_numpy(host.view(np.int64)).to(f"cuda:{device}")
            zipf_ptr = self.table.data_ptr()
        self.struct = InsertStream(spec.seed, spec.fresh_prefix, spec.dup_num, spec.dup_den,
                                   spec.dup_sel_seed, zipf_ptr, spec.zipf_n)


def _stream(device):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def gen_inserts(handle: StreamHandle, start: int, n: int, out: "torch.Tensor | None" = None,
                device: int = 0) -> "torch.Tensor":
    out = out if out is not None else torch.empty(n, dtype=torch.int64, device=f"cuda:{device}")
    check(_lib.lib().sbbf_gen_inserts(C.byref(handle.struct), start, n, C.c_void_p(out.data_ptr()),
                                      _stream(device)), "sbbf_gen_inserts")
    return out


def gen_lookups(handle: StreamHandle, lk: LookupSpec, num_inserts: int, start: int, n: int,
                out: "torch.Tensor | None" = None, device: int = 0) -> "torch.Tensor":
    out = out if out is not None else torch.empty(n, dtype=torch.int64, device=f"cuda:{device}")
    if lk.members_first:
        # positions [0, num_inserts) are the members in insert order
        m_end = min(max(num_inserts - start, 0), n)
        if m_end > 0:
            gen_inserts(handle, start, m_end, out[:m_end], device)
        if n - m_end > 0:
            nm = StreamHandle(InsertSpec(seed=lk.nonmember_seed, n=0), device)
            gen_inserts(nm, max(start - num_inserts, 0), n - m_end, out[m_end:], device)
        return out
    check(_lib.lib().sbbf_gen_lookups(C.byref(handle.struct), num_inserts, lk.nonmember_seed,
                                      lk.sel_seed, lk.p, lk.q, start, n,
                                      C.c_void_p(out.data_ptr()), _stream(device)),
          "sbbf_gen_lookups")
    return out


def member_count(lk: LookupSpec, num_inserts: int, start: int, n: int) -> int:
    """Members among lookup positions [start, start+n) (exact-fraction rule)."""
    if lk.members_first:
        return max(0, min(start + n, num_inserts) - min(start, num_inserts))
    return (start + n) * lk.p // lk.q - start * lk.p // lk.q
