"""TEST INFRASTRUCTURE ONLY — Python view of the CPU oracle.

Two checkers live here:

* ``Oracle``    — the plain-C restatement (``oracle/sbbf_oracle.c`` →
  ``oracle/liboracle.so``) of the reference's hot path
  (``/root/reference/proj/core/src/filter.cpp``) plus the workload streams.
* ``Reference`` — the reference's own core compiled unmodified
  (``oracle/_ref/libsbbf_ref.so``, built by ``oracle/Makefile`` from
  ``/root/reference``), used to pin ``Oracle`` and as bench.py's CPU baseline.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs import this package. The product
(``paper_2101_01719_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsbbf_ref.so")
REF_SRC = "/root/reference/proj/core/src"

LANE_SEEDS = (0x44974D91, 0x47B6137B, 0xA2B7289D, 0x8824AD5B,
              0x2DF1424B, 0x705495C7, 0x5C6BFB31, 0x9EFC4947)

_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)


def build(force: bool = False) -> None:
    """Compile the checkers (make -C oracle). The reference half is built only
    where /root/reference exists; elsewhere a prebuilt _ref/ is kept."""
    if force or not os.path.exists(ORACLE_SO) or (os.path.isdir(REF_SRC) and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


class Oracle:
    """ctypes wrapper of liboracle.so (the C restatement)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.oracle_block_index.restype = C.c_uint64
        L.oracle_block_index.argtypes = [C.c_uint64, C.c_uint64]
        L.oracle_make_mask.argtypes = [C.c_uint64, _u32p]
        L.oracle_add_hashes.argtypes = [_u32p, C.c_uint64, _u64p, C.c_uint64]
        L.oracle_find_hashes.argtypes = [_u32p, C.c_uint64, _u64p, C.c_uint64, _u8p]
        L.oracle_find_hashes_mt.argtypes = [_u32p, C.c_uint64, _u64p, C.c_uint64, _u8p, C.c_int]
        L.oracle_find_bits.argtypes = [_u32p, C.c_uint64, _u64p, C.c_uint64, _u32p]
        L.oracle_crc32_ieee.restype = C.c_uint32
        L.oracle_crc32_ieee.argtypes = [_u8p, C.c_uint64]
        L.oracle_image_size.restype = C.c_uint64
        L.oracle_image_size.argtypes = [C.c_uint64]
        L.oracle_serialize.restype = C.c_uint64
        L.oracle_serialize.argtypes = [_u32p, C.c_uint64, C.c_uint32, _u8p, C.c_uint64]
        L.oracle_image_crc.restype = C.c_uint32
        L.oracle_image_crc.argtypes = [_u32p, C.c_uint64, C.c_uint32]
        L.oracle_deserialize.restype = C.c_int
        L.oracle_deserialize.argtypes = [_u8p, C.c_uint64, _u64p, _u32p, _u32p]
        L.oracle_popcount_blocks.restype = C.c_uint64
        L.oracle_popcount_blocks.argtypes = [_u32p, C.c_uint64]
        L.oracle_splitmix64_at.restype = C.c_uint64
        L.oracle_splitmix64_at.argtypes = [C.c_uint64, C.c_uint64]
        L.oracle_gen_splitmix.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u64p]
        L.oracle_gen_mixed.argtypes = [C.c_uint64] * 8 + [_u64p]
        L.oracle_mt19937_64.argtypes = [C.c_uint64, C.c_uint64, _u64p]
        L.oracle_insert_value.restype = C.c_uint64
        L.oracle_insert_value.argtypes = [C.c_void_p, C.c_uint64]
        L.oracle_gen_inserts.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, _u64p]
        L.oracle_gen_lookups.argtypes = [C.c_void_p] + [C.c_uint64] * 7 + [_u64p]
        L.oracle_xxh64.restype = C.c_uint64
        L.oracle_xxh64.argtypes = [_u8p, C.c_uint64, C.c_uint64]

    # -- hot path --------------------------------------------------------
    def block_index(self, h: int, nb: int) -> int:
        return int(self.lib.oracle_block_index(h, nb))

    def make_mask(self, h: int) -> list[int]:
        out = np.zeros(8, np.uint32)
        self.lib.oracle_make_mask(h, _p(out, _u32p))
        return [int(x) for x in out]

    def new_blocks(self, nb: int) -> np.ndarray:
        return np.zeros((nb, 8), np.uint32)

    def add_hashes(self, blocks: np.ndarray, hashes) -> None:
        h = _u64(hashes)
        self.lib.oracle_add_hashes(_p(blocks, _u32p), blocks.shape[0], _p(h, _u64p), h.size)

    def build(self, nb: int, hashes) -> np.ndarray:
        b = self.new_blocks(nb)
        self.add_hashes(b, hashes)
        return b

    def find_hashes(self, blocks: np.ndarray, hashes, threads: int = 1) -> np.ndarray:
        h = _u64(hashes)
        out = np.empty(h.size, np.uint8)
        self.lib.oracle_find_hashes_mt(_p(blocks, _u32p), blocks.shape[0], _p(h, _u64p), h.size,
                                       _p(out, _u8p), threads)
        return out

    def find_bits(self, blocks: np.ndarray, hashes) -> np.ndarray:
        h = _u64(hashes)
        out = np.empty((h.size + 31) // 32, np.uint32)
        self.lib.oracle_find_bits(_p(blocks, _u32p), blocks.shape[0], _p(h, _u64p), h.size,
                                  _p(out, _u32p))
        return out

    # -- image -----------------------------------------------------------
    def crc32(self, data: bytes) -> int:
        a = np.frombuffer(data, np.uint8) if len(data) else np.zeros(1, np.uint8)
        return int(self.lib.oracle_crc32_ieee(_p(a, _u8p), len(data)))

    def serialize(self, blocks: np.ndarray, hasher_id: int = 0) -> bytes:
        nb = blocks.shape[0]
        out = np.empty(int(self.lib.oracle_image_size(nb)), np.uint8)
        n = self.lib.oracle_serialize(_p(blocks, _u32p), nb, hasher_id, _p(out, _u8p), out.size)
        assert n == out.size
        return out.tobytes()

    def image_crc(self, blocks: np.ndarray, hasher_id: int = 0) -> int:
        return int(self.lib.oracle_image_crc(_p(blocks, _u32p), blocks.shape[0], hasher_id))

    def deserialize(self, data: bytes):
        """Returns (errcode, blocks, hasher_id); errcode 0 = ok, else 1+PersistErrc."""
        a = np.frombuffer(data, np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
        nb = C.c_uint64(0)
        hid = C.c_uint32(0)
        rc = self.lib.oracle_deserialize(_p(a, _u8p), len(data), C.byref(nb), C.byref(hid), None)
        if rc:
            return rc, None, None
        blocks = np.zeros((nb.value, 8), np.uint32)
        self.lib.oracle_deserialize(_p(a, _u8p), len(data), C.byref(nb), C.byref(hid),
                                    _p(blocks, _u32p))
        return 0, blocks, hid.value

    def popcount(self, blocks: np.ndarray) -> int:
        return int(self.lib.oracle_popcount_blocks(_p(blocks, _u32p), blocks.shape[0]))

    # -- streams ---------------------------------------------------------
    def splitmix(self, seed: int, start: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint64)
        self.lib.oracle_gen_splitmix(seed, start, n, _p(out, _u64p))
        return out

    def mixed(self, member_seed, num_members, nonmember_seed, sel_seed, p, q, start, n):
        out = np.empty(n, np.uint64)
        self.lib.oracle_gen_mixed(member_seed, num_members, nonmember_seed, sel_seed, p, q,
                                  start, n, _p(out, _u64p))
        return out

    def stream(self, spec, zipf_table=None) -> "OracleStream":
        """Host insert stream for a workload InsertSpec (config 4 needs the table)."""
        return OracleStream(spec, zipf_table)

    def gen_inserts(self, st: "OracleStream", start: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint64)
        self.lib.oracle_gen_inserts(C.byref(st.struct), start, n, _p(out, _u64p))
        return out

    def gen_lookups(self, st: "OracleStream", lk, num_inserts: int, start: int, n: int) -> np.ndarray:
        """Mirror of paper_2101_01719_b200.workload.gen_lookups on the host."""
        if lk.members_first:
            m_end = min(max(num_inserts - start, 0), n)
            parts = []
            if m_end > 0:
                parts.append(self.gen_inserts(st, start, m_end))
            if n - m_end > 0:
                parts.append(self.splitmix(lk.nonmember_seed, max(start - num_inserts, 0), n - m_end))
            return np.concatenate(parts) if parts else np.zeros(0, np.uint64)
        out = np.empty(n, np.uint64)
        self.lib.oracle_gen_lookups(C.byref(st.struct), num_inserts, lk.nonmember_seed, lk.sel_seed,
                                    lk.p, lk.q, start, n, _p(out, _u64p))
        return out

    def mt19937_64(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint64)
        self.lib.oracle_mt19937_64(seed, n, _p(out, _u64p))
        return out

    def xxh64(self, data: bytes, seed: int = 0) -> int:
        a = np.frombuffer(data, np.uint8) if len(data) else np.zeros(1, np.uint8)
        return int(self.lib.oracle_xxh64(_p(a, _u8p), len(data), seed))


class _StreamStruct(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("fresh_prefix", C.c_uint64), ("dup_num", C.c_uint64),
                ("dup_den", C.c_uint64), ("dup_sel_seed", C.c_uint64), ("zipf_cdf", C.c_void_p),
                ("zipf_n", C.c_uint64)]


class OracleStream:
    def __init__(self, spec, zipf_table=None):
        self.table = None
        ptr = None
        if spec.dup_num:
            self.table = np.ascontiguousarray(zipf_table, np.uint64)
            assert self.table.size == spec.zipf_n
            ptr = self.table.ctypes.data
        self.struct = _StreamStruct(spec.seed, spec.fresh_prefix, spec.dup_num, spec.dup_den,
                                    spec.dup_sel_seed, ptr, spec.zipf_n)


class Reference:
    """ctypes wrapper of oracle/_ref/libsbbf_ref.so (the reference itself)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (reference sources absent)")
        L = self.lib = C.CDLL(path)
        L.ref_block_index.restype = C.c_uint64
        L.ref_block_index.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_make_mask.argtypes = [C.c_uint64, _u32p]
        L.ref_vector_backend_available.restype = C.c_int
        L.ref_filter_new.restype = C.c_void_p
        L.ref_filter_new.argtypes = [C.c_uint64, C.c_uint32, C.c_int]
        L.ref_filter_free.argtypes = [C.c_void_p]
        L.ref_filter_add.argtypes = [C.c_void_p, _u64p, C.c_uint64]
        L.ref_filter_add_one.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_filter_find_one.restype = C.c_int
        L.ref_filter_find_one.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_filter_find.argtypes = [C.c_void_p, _u64p, C.c_uint64, _u8p]
        L.ref_filter_find_mt.argtypes = [C.c_void_p, _u64p, C.c_uint64, _u8p, C.c_int]
        L.ref_filter_num_buckets.restype = C.c_uint64
        L.ref_filter_num_buckets.argtypes = [C.c_void_p]
        L.ref_filter_blocks.argtypes = [C.c_void_p, _u32p]
        L.ref_filter_from_blocks.restype = C.c_void_p
        L.ref_filter_from_blocks.argtypes = [_u32p, C.c_uint64, C.c_uint32]
        L.ref_filter_serialize.restype = C.c_uint64
        L.ref_filter_serialize.argtypes = [C.c_void_p, _u8p, C.c_uint64]
        L.ref_deserialize.restype = C.c_int
        L.ref_deserialize.argtypes = [_u8p, C.c_uint64, C.POINTER(C.c_void_p)]
        L.ref_crc32.restype = C.c_uint32
        L.ref_crc32.argtypes = [_u8p, C.c_uint64]
        L.ref_hash_key.restype = C.c_uint64
        L.ref_hash_key.argtypes = [_u8p, C.c_uint64, C.c_uint64]
        L.ref_hash_u64_key.restype = C.c_uint64
        L.ref_hash_u64_key.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_mt19937_64.argtypes = [C.c_uint64, C.c_uint64, _u64p]
        L.ref_fpp_sim.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _u64p,
                                  C.POINTER(C.c_uint32)]
        L.ref_sbbf_fpp.restype = C.c_double
        L.ref_sbbf_fpp.argtypes = [C.c_double]
        L.ref_standard_bloom_fpp.restype = C.c_double
        L.ref_standard_bloom_fpp.argtypes = [C.c_double, C.c_uint]
        L.ref_optimal_bloom_k.restype = C.c_uint
        L.ref_optimal_bloom_k.argtypes = [C.c_double]
        L.ref_size_for.restype = C.c_uint64
        L.ref_size_for.argtypes = [C.c_uint64, C.c_double]
        L.ref_time_build_probe.argtypes = [C.c_uint64, _u64p, C.c_uint64, _u64p, C.c_uint64, _u8p,
                                           C.c_int, C.c_int, C.POINTER(C.c_double),
                                           C.POINTER(C.c_double), C.POINTER(C.c_void_p)]

    def block_index(self, h: int, nb: int) -> int:
        return int(self.lib.ref_block_index(h, nb))

    def make_mask(self, h: int) -> list[int]:
        out = np.zeros(8, np.uint32)
        self.lib.ref_make_mask(h, _p(out, _u32p))
        return [int(x) for x in out]

    def filter(self, nb: int, hasher_id: int = 0, backend: int = 0) -> "RefFilter":
        return RefFilter(self, nb, hasher_id, backend)

    def build(self, nb: int, hashes) -> np.ndarray:
        f = self.filter(nb)
        f.add_hashes(hashes)
        return f.blocks()

    def mt19937_64(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint64)
        self.lib.ref_mt19937_64(seed, n, _p(out, _u64p))
        return out

    def fpp_sim(self, ndv: int, filter_bytes: int, queries: int, seed: int):
        """(false positives, image CRC) of the reference's run_fpp_sim loop."""
        fp = C.c_uint64(0)
        crc = C.c_uint32(0)
        self.lib.ref_fpp_sim(ndv, filter_bytes // 32, queries, seed, C.byref(fp), C.byref(crc))
        return int(fp.value), int(crc.value)

    def crc32(self, data: bytes) -> int:
        a = np.frombuffer(data, np.uint8) if len(data) else np.zeros(1, np.uint8)
        return int(self.lib.ref_crc32(_p(a, _u8p), len(data)))

    def hash_key(self, data: bytes, seed: int = 0) -> int:
        a = np.frombuffer(data, np.uint8) if len(data) else np.zeros(1, np.uint8)
        return int(self.lib.ref_hash_key(_p(a, _u8p), len(data), seed))

    def deserialize_code(self, data: bytes) -> int:
        a = np.frombuffer(data, np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
        out = C.c_void_p()
        rc = self.lib.ref_deserialize(_p(a, _u8p), len(data), C.byref(out))
        if rc == 0:
            self.lib.ref_filter_free(out)
        return rc

    def time_build_probe(self, nb, inserts, lookups, threads=1, reps=3):
        """run_bench's timing (tools/harness.cpp:160-201). Returns
        (insert_seconds[reps], lookup_seconds[reps], results u8, blocks)."""
        ins, look = _u64(inserts), _u64(lookups)
        res = np.empty(look.size, np.uint8)
        ti = (C.c_double * reps)()
        tl = (C.c_double * reps)()
        keep = C.c_void_p()
        self.lib.ref_time_build_probe(nb, _p(ins, _u64p), ins.size, _p(look, _u64p), look.size,
                                      _p(res, _u8p), threads, reps, ti, tl, C.byref(keep))
        blocks = np.zeros((nb, 8), np.uint32)
        self.lib.ref_filter_blocks(keep, _p(blocks, _u32p))
        self.lib.ref_filter_free(keep)
        return list(ti), list(tl), res, blocks


class RefFilter:
    def __init__(self, ref: Reference, nb: int, hasher_id: int = 0, backend: int = 0):
        self.ref = ref
        self.h = ref.lib.ref_filter_new(nb, hasher_id, backend)
        if not self.h:
            raise ValueError("reference SplitBlockFilter constructor threw")
        self.nb = nb

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_filter_free(self.h)
            self.h = None

    def add_hashes(self, hashes) -> None:
        h = _u64(hashes)
        self.ref.lib.ref_filter_add(self.h, _p(h, _u64p), h.size)

    def add_hash(self, h: int) -> None:
        self.ref.lib.ref_filter_add_one(self.h, h)

    def find_hash(self, h: int) -> bool:
        return bool(self.ref.lib.ref_filter_find_one(self.h, h))

    def find_hashes(self, hashes, threads: int = 1) -> np.ndarray:
        h = _u64(hashes)
        out = np.empty(h.size, np.uint8)
        self.ref.lib.ref_filter_find_mt(self.h, _p(h, _u64p), h.size, _p(out, _u8p), threads)
        return out

    def blocks(self) -> np.ndarray:
        b = np.zeros((self.nb, 8), np.uint32)
        self.ref.lib.ref_filter_blocks(self.h, _p(b, _u32p))
        return b

    def serialize(self) -> bytes:
        out = np.empty(17 + 32 * self.nb + 4, np.uint8)
        n = self.ref.lib.ref_filter_serialize(self.h, _p(out, _u8p), out.size)
        assert n == out.size
        return out.tobytes()


def bits_to_bytes(bits: np.ndarray, n: int) -> np.ndarray:
    """Unpack an LSB-first bitmap (bit k%32 of word k//32) to 0/1 bytes."""
    return np.unpackbits(np.ascontiguousarray(bits, np.uint32).view(np.uint8),
                         bitorder="little")[:n]
