"""Host-side mirror of the reference's ``sbbf::SplitBlockFilter`` over the C ABI.

Reference interface: ``/root/reference/proj/core/include/sbbf/filter.hpp:65-109``
(names, argument meaning and error behaviour are kept):

===========================  ==========================================  =========================
reference (filter.hpp)       here                                        C ABI (include/sbbf_gpu.h)
===========================  ==========================================  =========================
ctor(num_buckets, hasher_id)  ``SplitBlockFilter(num_buckets, hasher_id)``  ``sbbf_gpu_create``
  throws invalid_argument     raises ``ValueError`` for 0 buckets
from_blocks(blocks, id)       ``SplitBlockFilter.from_blocks``            ``sbbf_gpu_from_host``
add_hash / find_hash          ``add_hash`` / ``find_hash``                ``sbbf_gpu_add_hash`` ...
add_hashes(span)              ``add_hashes(hashes)``                      ``sbbf_gpu_insert_batch`` (device)
                                                                          ``sbbf_gpu_add_hashes_host`` (host)
find_hashes(span, uint8_t*)   ``find_hashes(hashes, results=None)``      ``sbbf_gpu_find_batch`` / ``_host``
(packed bitmap, new)          ``find_hashes_bits(hashes, out=None)``      ``sbbf_gpu_find_batch_bits``
num_buckets/size_bytes        properties-as-methods, same names
blocks()                      ``blocks()`` -> (num_buckets, 8) uint32      ``sbbf_gpu_to_host``
hasher_id/set_hasher_id       same                                        ``sbbf_gpu_{set_,}hasher_id``
operator==                    ``__eq__`` (same blocks and hasher id)
===========================  ==========================================  =========================

``hashes`` may be a CUDA ``torch.Tensor`` (int64/uint64, on the filter's
device; the call is asynchronous on torch's current stream) or any host
array-like of uint64 (numpy, list, CPU tensor; the call is synchronous and
pipelines the host<->device copies).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check

try:  # torch is plumbing (device memory, streams); host arrays work without it
    import torch
except ImportError:  # pragma: no cover
    torch = None


PERSIST_ERRC = {1: "kTruncated", 2: "kBadMagic", 3: "kBadVersion", 4: "kBadBucketCount",
                5: "kBadChecksum", 6: "kIo"}  # persist.hpp:33-40 (value + 1)


class PersistError(ValueError):
    """PersistError (persist.hpp:42-51): .code is the PersistErrc name."""

    def __init__(self, errc: int, what: str):
        super().__init__(what)
        self.errc = errc
        self.code = PERSIST_ERRC.get(errc, str(errc))


def _is_cuda_tensor(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def _host_u64(x) -> np.ndarray:
    if torch is not None and isinstance(x, torch.Tensor):
        x = x.detach().cpu().numpy()
    a = np.asarray(x)
    if a.dtype != np.uint64:
        a = a.astype(np.uint64) if a.size else np.zeros(0, np.uint64)
    return np.ascontiguousarray(a.reshape(-1))


def _dev_u64(t) -> "torch.Tensor":
    if t.dtype not in (torch.int64, torch.uint64):
        raise TypeError(f"hash tensor must be int64/uint64, got {t.dtype}")
    return t.contiguous().view(-1)


def _stream_ptr(device: int):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class SplitBlockFilter:
    """B200 split block Bloom filter, byte-compatible with the reference."""

    def __init__(self, num_buckets: int, hasher_id: int = 0, device: int = 0):
        num_buckets = int(num_buckets)
        if num_buckets <= 0:
            # filter.cpp:160-162: std::invalid_argument
            raise ValueError("SplitBlockFilter needs at least one bucket")
        self._h = C.c_void_p()
        L = _lib.lib()
        check(L.sbbf_gpu_create(num_buckets, int(device), C.byref(self._h)), "sbbf_gpu_create")
        self._device = int(device)
        if hasher_id:
            check(L.sbbf_gpu_set_hasher_id(self._h, int(hasher_id)), "set_hasher_id")

    # -- lifetime ------------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            _lib.lib().sbbf_gpu_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self) -> "SplitBlockFilter":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    def __repr__(self) -> str:
        if not (getattr(self, "_h", None) and self._h.value):
            return "SplitBlockFilter(<closed>)"
        return (f"SplitBlockFilter(num_buckets={self.num_buckets()}, bytes={self.size_bytes()}, "
                f"hasher_id={self.hasher_id()}, device={self._device})")

    @classmethod
    def from_blocks(cls, blocks, hasher_id: int = 0, device: int = 0) -> "SplitBlockFilter":
        """filter.hpp:74-75 — adopt existing block contents ((B, 8) uint32 or B*32 bytes)."""
        b = np.ascontiguousarray(np.asarray(blocks).view(np.uint32).reshape(-1, 8))
        if b.shape[0] == 0:
            raise ValueError("SplitBlockFilter needs at least one bucket")
        f = cls(b.shape[0], hasher_id, device)
        check(_lib.lib().sbbf_gpu_from_host(f._h, b.ctypes.data_as(C.c_void_p), b.nbytes),
              "sbbf_gpu_from_host")
        return f

    def clear(self) -> None:
        """Zero all blocks (a fresh filter), stream-ordered on torch's current stream."""
        stream = _stream_ptr(self._device) if torch is not None and torch.cuda.is_available() else None
        check(_lib.lib().sbbf_gpu_clear(self._h, stream), "sbbf_gpu_clear")

    # -- accessors (filter.hpp:85-94) ------------------------------------------
    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @property
    def device(self) -> int:
        return self._device

    def num_buckets(self) -> int:
        return int(_lib.lib().sbbf_gpu_num_buckets(self._h))

    def size_bytes(self) -> int:
        return int(_lib.lib().sbbf_gpu_size_bytes(self._h))

    def hasher_id(self) -> int:
        return int(_lib.lib().sbbf_gpu_hasher_id(self._h))

    def set_hasher_id(self, hasher_id: int) -> None:
        check(_lib.lib().sbbf_gpu_set_hasher_id(self._h, int(hasher_id)), "set_hasher_id")

    def device_blocks_ptr(self) -> int:
        return int(_lib.lib().sbbf_gpu_device_blocks(self._h) or 0)

    def blocks(self) -> np.ndarray:
        """filter.hpp:87 — a host copy of the block array, shape (num_buckets, 8) uint32."""
        out = np.empty((self.num_buckets(), 8), np.uint32)
        check(_lib.lib().sbbf_gpu_to_host(self._h, out.ctypes.data_as(C.c_void_p), out.nbytes),
              "sbbf_gpu_to_host")
        return out

    def blocks_range(self, first: int, count: int) -> np.ndarray:
        """Host copy of blocks [first, first+count) — spot checks and shard gathers."""
        out = np.empty((int(count), 8), np.uint32)
        check(_lib.lib().sbbf_gpu_blocks_to_host(self._h, int(first), int(count),
                                                 out.ctypes.data_as(C.c_void_p)), "blocks_to_host")
        return out

    def __eq__(self, other) -> bool:
        """filter.hpp:97-101 — same blocks and same hasher id."""
        if not isinstance(other, SplitBlockFilter):
            return NotImplemented
        return self.hasher_id() == other.hasher_id() and np.array_equal(self.blocks(), other.blocks())

    __hash__ = None

    # -- tuning ------------------------------------------------------------------
    def set_insert_variant(self, v: int) -> None:
        check(_lib.lib().sbbf_gpu_set_insert_variant(self._h, int(v)), "set_insert_variant")

    def set_find_variant(self, v: int) -> None:
        check(_lib.lib().sbbf_gpu_set_find_variant(self._h, int(v)), "set_find_variant")

    def resolved_variants(self, n: int) -> tuple[int, int]:
        L = _lib.lib()
        return (int(L.sbbf_gpu_resolved_insert_variant(self._h, n)),
                int(L.sbbf_gpu_resolved_find_variant(self._h, n)))

    # -- hot path ----------------------------------------------------------------
    def add_hash(self, h: int) -> None:
        check(_lib.lib().sbbf_gpu_add_hash(self._h, int(h) & 0xFFFFFFFFFFFFFFFF), "add_hash")

    def find_hash(self, h: int) -> bool:
        found = C.c_int(0)
        check(_lib.lib().sbbf_gpu_find_hash(self._h, int(h) & 0xFFFFFFFFFFFFFFFF, C.byref(found)),
              "find_hash")
        return bool(found.value)

    def add_hashes(self, hashes) -> None:
        """filter.hpp:81 — element-wise add_hash over the batch."""
        L = _lib.lib()
        if _is_cuda_tensor(hashes):
            t = _dev_u64(hashes)
            check(L.sbbf_gpu_insert_batch(self._h, C.c_void_p(t.data_ptr()), t.numel(),
                                          _stream_ptr(self._device)), "sbbf_gpu_insert_batch")
            return
        a = _host_u64(hashes)
        check(L.sbbf_gpu_add_hashes_host(self._h, a.ctypes.data_as(C.c_void_p), a.size),
              "sbbf_gpu_add_hashes_host")

    def find_hashes(self, hashes, results=None):
        """filter.hpp:82-83 — one 0/1 byte per key. Device in -> device out."""
        L = _lib.lib()
        if _is_cuda_tensor(hashes):
            t = _dev_u64(hashes)
            out = results if results is not None else torch.empty(t.numel(), dtype=torch.uint8,
                                                                  device=t.device)
            check(L.sbbf_gpu_find_batch(self._h, C.c_void_p(t.data_ptr()), t.numel(),
                                        C.c_void_p(out.data_ptr()), _stream_ptr(self._device)),
                  "sbbf_gpu_find_batch")
            return out
        a = _host_u64(hashes)
        out = results if results is not None else np.empty(a.size, np.uint8)
        check(L.sbbf_gpu_find_hashes_host(self._h, a.ctypes.data_as(C.c_void_p), a.size,
                                          out.ctypes.data_as(C.c_void_p)), "sbbf_gpu_find_hashes_host")
        return out

    def find_hashes_bits(self, hashes, out=None):
        """Packed answers: bit k%32 of word k//32 (uint32, LSB first) is key k."""
        L = _lib.lib()
        if _is_cuda_tensor(hashes):
            t = _dev_u64(hashes)
            nwords = (t.numel() + 31) // 32
            o = out if out is not None else torch.empty(nwords, dtype=torch.int32, device=t.device)
            check(L.sbbf_gpu_find_batch_bits(self._h, C.c_void_p(t.data_ptr()), t.numel(),
                                             C.c_void_p(o.data_ptr()), _stream_ptr(self._device)),
                  "sbbf_gpu_find_batch_bits")
            return o
        a = _host_u64(hashes)
        o = out if out is not None else np.empty((a.size + 31) // 32, np.uint32)
        check(L.sbbf_gpu_find_bits_host(self._h, a.ctypes.data_as(C.c_void_p), a.size,
                                        o.ctypes.data_as(C.c_void_p)), "sbbf_gpu_find_bits_host")
        return o

    # -- FilterImage v1 (persist.hpp:14-66, persist.cpp:72-157) ----------------------
    def image_crc(self) -> int:
        """The image trailer CRC-32 (computed on the GPU)."""
        crc = C.c_uint32(0)
        check(_lib.lib().sbbf_gpu_image_crc(self._h, C.byref(crc)), "sbbf_gpu_image_crc")
        return int(crc.value)

    def blocks_crc(self) -> int:
        """CRC-32 of the block array bytes alone (GPU): a shard's part of the
        gathered image CRC (ShardedFilter.image_crc combines them)."""
        crc = C.c_uint32(0)
        check(_lib.lib().sbbf_gpu_blocks_crc(self._h, C.byref(crc)), "sbbf_gpu_blocks_crc")
        return int(crc.value)

    def serialize(self) -> bytes:
        """serialize() (persist.cpp:72-88): the canonical v1 image."""
        L = _lib.lib()
        out = np.empty(int(L.sbbf_gpu_image_size(self.num_buckets())), np.uint8)
        written = C.c_uint64(0)
        check(L.sbbf_gpu_serialize(self._h, out.ctypes.data_as(C.c_void_p), out.size, C.byref(written)),
              "sbbf_gpu_serialize")
        return out.tobytes()

    @classmethod
    def _adopt(cls, h: C.c_void_p, device: int) -> "SplitBlockFilter":
        f = cls.__new__(cls)
        f._h = h
        f._device = device
        return f

    @classmethod
    def deserialize(cls, image: bytes, device: int = 0) -> "SplitBlockFilter":
        """deserialize() (persist.cpp:90-126); raises PersistError with the
        reference's error code on malformed images."""
        a = np.frombuffer(image, np.uint8) if len(image) else np.zeros(1, np.uint8)
        h = C.c_void_p()
        errc = C.c_int(0)
        rc = _lib.lib().sbbf_gpu_deserialize(a.ctypes.data_as(C.c_void_p), len(image), device, C.byref(h),
                                             C.byref(errc))
        if rc == _lib.SBBF_EFORMAT:
            raise PersistError(errc.value, _lib.last_error())
        check(rc, "sbbf_gpu_deserialize")
        return cls._adopt(h, device)

    def save(self, path: str) -> None:
        """save_filter (persist.cpp:128-142)."""
        errc = C.c_int(0)
        rc = _lib.lib().sbbf_gpu_save(self._h, str(path).encode(), C.byref(errc))
        if rc == _lib.SBBF_EFORMAT:
            raise PersistError(errc.value, _lib.last_error())
        check(rc, "sbbf_gpu_save")

    @classmethod
    def load(cls, path: str, device: int = 0) -> "SplitBlockFilter":
        """load_filter (persist.cpp:144-157)."""
        h = C.c_void_p()
        errc = C.c_int(0)
        rc = _lib.lib().sbbf_gpu_load(str(path).encode(), device, C.byref(h), C.byref(errc))
        if rc == _lib.SBBF_EFORMAT:
            raise PersistError(errc.value, _lib.last_error())
        check(rc, "sbbf_gpu_load")
        return cls._adopt(h, device)

    # -- XXH64 key frontend (kHasherXxh64, hash.hpp:12): u64 keys hashed in-kernel --
    def _dev_keys(self, keys):
        if _is_cuda_tensor(keys):
            return _dev_u64(keys)
        a = _host_u64(keys)
        return torch.from_numpy(a.view(np.int64)).to(torch.device("cuda", self._device))

    def add_keys(self, keys, seed: int = 0) -> None:
        """Insert u64 keys hashed with hash_u64_key(key, seed) (hash.cpp:108-114)."""
        t = self._dev_keys(keys)
        check(_lib.lib().sbbf_gpu_insert_keys_u64(self._h, C.c_void_p(t.data_ptr()), t.numel(), seed,
                                                  _stream_ptr(self._device)), "sbbf_gpu_insert_keys_u64")

    def find_keys(self, keys, seed: int = 0, results=None):
        t = self._dev_keys(keys)
        out = results if results is not None else torch.empty(t.numel(), dtype=torch.uint8, device=t.device)
        check(_lib.lib().sbbf_gpu_find_keys_u64(self._h, C.c_void_p(t.data_ptr()), t.numel(), seed,
                                                C.c_void_p(out.data_ptr()), _stream_ptr(self._device)),
              "sbbf_gpu_find_keys_u64")
        return out

    def find_keys_bits(self, keys, seed: int = 0, out=None):
        t = self._dev_keys(keys)
        o = out if out is not None else torch.empty((t.numel() + 31) // 32, dtype=torch.int32, device=t.device)
        check(_lib.lib().sbbf_gpu_find_keys_u64_bits(self._h, C.c_void_p(t.data_ptr()), t.numel(), seed,
                                                     C.c_void_p(o.data_ptr()), _stream_ptr(self._device)),
              "sbbf_gpu_find_keys_u64_bits")
        return o


def hash_u64_keys(keys: "torch.Tensor", seed: int = 0) -> "torch.Tensor":
    """hash_u64_key (hash.cpp:108-114) on device: XXH64 of each key's 8 LE bytes."""
    t = _dev_u64(keys)
    out = torch.empty(t.numel(), dtype=torch.int64, device=t.device)
    check(_lib.lib().sbbf_gpu_hash_u64_keys(C.c_void_p(t.data_ptr()), t.numel(), seed,
                                            C.c_void_p(out.data_ptr()), _stream_ptr(t.device.index or 0)),
          "sbbf_gpu_hash_u64_keys")
    return out


def hash_keys(keys, seed: int = 0, device: int = 0) -> "torch.Tensor":
    """hash_key (hash.cpp:100-106) on device for a list of byte strings."""
    blobs = [k.encode() if isinstance(k, str) else bytes(k) for k in keys]
    offsets = np.zeros(len(blobs) + 1, np.uint64)
    offsets[1:] = np.cumsum([len(b) for b in blobs], dtype=np.uint64)
    dev = torch.device("cuda", device)
    data = torch.frombuffer(bytearray(b"".join(blobs)) or bytearray(1), dtype=torch.uint8).to(dev)
    offs = torch.from_numpy(offsets.view(np.int64)).to(dev)
    out = torch.empty(len(blobs), dtype=torch.int64, device=dev)
    check(_lib.lib().sbbf_gpu_hash_bytes(C.c_void_p(data.data_ptr()), C.c_void_p(offs.data_ptr()), len(blobs),
                                         seed, C.c_void_p(out.data_ptr()), _stream_ptr(device)),
          "sbbf_gpu_hash_bytes")
    return out


def hash_counter_strings(start: int, n: int, seed: int = 0, device: int = 0) -> "torch.Tensor":
    """hash_key(std::to_string(c)) for c in [start, start + n) on device — the
    reference's byte-string experiment keys (harness.cpp:60-65)."""
    dev = torch.device("cuda", device)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    check(_lib.lib().sbbf_gpu_hash_counter_strings(start, n, seed, C.c_void_p(out.data_ptr()) if n else None,
                                                   _stream_ptr(device)), "sbbf_gpu_hash_counter_strings")
    return out


def block_index_batch(hashes: "torch.Tensor", num_buckets: int) -> "torch.Tensor":
    """filter.hpp:42 on device, for known-answer tests."""
    t = _dev_u64(hashes)
    out = torch.empty(t.numel(), dtype=torch.int64, device=t.device)
    check(_lib.lib().sbbf_gpu_block_index_batch(C.c_void_p(t.data_ptr()), t.numel(), int(num_buckets),
                                                C.c_void_p(out.data_ptr()),
                                                _stream_ptr(t.device.index or 0)), "block_index_batch")
    return out


def make_mask_batch(hashes: "torch.Tensor") -> "torch.Tensor":
    """filter.hpp:47 on device: (n, 8) lane masks (int32 view of uint32)."""
    t = _dev_u64(hashes)
    out = torch.empty((t.numel(), 8), dtype=torch.int32, device=t.device)
    check(_lib.lib().sbbf_gpu_make_mask_batch(C.c_void_p(t.data_ptr()), t.numel(),
                                              C.c_void_p(out.data_ptr()),
                                              _stream_ptr(t.device.index or 0)), "make_mask_batch")
    return out
