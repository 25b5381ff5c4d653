"""ctypes binding of ``libsbbf_gpu.so`` (the C ABI in ``include/sbbf_gpu.h``).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2101_01719_b200/csrc``). There is deliberately no fallback:
if the library is missing or no CUDA device is usable, every entry point
raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# SBBF_LIB=<tag> selects libsbbf_gpu_<tag>.so: `debug` (device-side bounds
# checks, `make debug`) or an A/B build (`make exp EXP_FLAGS=...`)
_TAG = os.environ.get("SBBF_LIB", "")
LIB_PATH = os.path.join(HERE, f"libsbbf_gpu_{_TAG}.so" if _TAG else "libsbbf_gpu.so")

SBBF_OK = 0
SBBF_EINVAL = -1
SBBF_ENOMEM = -2
SBBF_ECUDA = -3
SBBF_ENODEV = -4
SBBF_EFORMAT = -5

(INSERT_AUTO, INSERT_LANE8, INSERT_LANE8_TEST, INSERT_THREAD, INSERT_WIDE, INSERT_WIDE_TEST,
 INSERT_BLOCKED) = range(7)
FIND_AUTO, FIND_GLOBAL, FIND_SMEM, FIND_BLOCKED = range(4)

# Every symbol include/sbbf_gpu.h and include/sbbf_workload.h declare, with
# (restype, argtypes). tests/test_abi.py checks the .so exports all of them.
_vp, _u64, _u32, _i = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
_u64p = C.POINTER(C.c_uint64)
PROTOTYPES = {
    "sbbf_gpu_create": (_i, [_u64, _i, C.POINTER(_vp)]),
    "sbbf_gpu_destroy": (_i, [_vp]),
    "sbbf_gpu_clear": (_i, [_vp, _vp]),
    "sbbf_gpu_num_buckets": (_u64, [_vp]),
    "sbbf_gpu_size_bytes": (_u64, [_vp]),
    "sbbf_gpu_hasher_id": (_u32, [_vp]),
    "sbbf_gpu_set_hasher_id": (_i, [_vp, _u32]),
    "sbbf_gpu_device": (_i, [_vp]),
    "sbbf_gpu_device_blocks": (_vp, [_vp]),
    "sbbf_gpu_insert_batch": (_i, [_vp, _vp, _u64, _vp]),
    "sbbf_gpu_find_batch": (_i, [_vp, _vp, _u64, _vp, _vp]),
    "sbbf_gpu_find_batch_bits": (_i, [_vp, _vp, _u64, _vp, _vp]),
    "sbbf_gpu_add_hashes_host": (_i, [_vp, _vp, _u64]),
    "sbbf_gpu_find_hashes_host": (_i, [_vp, _vp, _u64, _vp]),
    "sbbf_gpu_find_bits_host": (_i, [_vp, _vp, _u64, _vp]),
    "sbbf_gpu_add_hash": (_i, [_vp, _u64]),
    "sbbf_gpu_find_hash": (_i, [_vp, _u64, C.POINTER(_i)]),
    "sbbf_gpu_to_host": (_i, [_vp, _vp, _u64]),
    "sbbf_gpu_from_host": (_i, [_vp, _vp, _u64]),
    "sbbf_gpu_blocks_to_host": (_i, [_vp, _u64, _u64, _vp]),
    "sbbf_gpu_block_index_batch": (_i, [_vp, _u64, _u64, _vp, _vp]),
    "sbbf_gpu_make_mask_batch": (_i, [_vp, _u64, _vp, _vp]),
    "sbbf_gpu_block_index_host": (_i, [_vp, _u64, _u64, _vp, _i]),
    "sbbf_gpu_make_mask_host": (_i, [_vp, _u64, _vp, _i]),
    "sbbf_gpu_set_insert_variant": (_i, [_vp, _i]),
    "sbbf_gpu_release_scratch": (_i, [_vp]),
    "sbbf_gpu_set_find_variant": (_i, [_vp, _i]),
    "sbbf_gpu_resolved_insert_variant": (_i, [_vp, _u64]),
    "sbbf_gpu_resolved_find_variant": (_i, [_vp, _u64]),
    "sbbf_gpu_set_l2_fetch_granularity": (_i, [_i, _i, C.POINTER(_i)]),
    "sbbf_gpu_image_size": (_u64, [_u64]),
    "sbbf_gpu_image_crc": (_i, [_vp, C.POINTER(_u32)]),
    "sbbf_gpu_blocks_crc": (_i, [_vp, C.POINTER(_u32)]),
    "sbbf_crc32_update": (_u32, [_u32, _vp, _u64]),
    "sbbf_crc32_combine": (_u32, [_u32, _u32, _u64]),
    "sbbf_gpu_serialize": (_i, [_vp, _vp, _u64, C.POINTER(_u64)]),
    "sbbf_gpu_deserialize": (_i, [_vp, _u64, _i, C.POINTER(_vp), C.POINTER(_i)]),
    "sbbf_gpu_save": (_i, [_vp, C.c_char_p, C.POINTER(_i)]),
    "sbbf_gpu_load": (_i, [C.c_char_p, _i, C.POINTER(_vp), C.POINTER(_i)]),
    "sbbf_gpu_hash_u64_keys": (_i, [_vp, _u64, _u64, _vp, _vp]),
    "sbbf_gpu_hash_bytes": (_i, [_vp, _vp, _u64, _u64, _vp, _vp]),
    "sbbf_gpu_insert_keys_u64": (_i, [_vp, _vp, _u64, _u64, _vp]),
    "sbbf_gpu_find_keys_u64": (_i, [_vp, _vp, _u64, _u64, _vp, _vp]),
    "sbbf_gpu_find_keys_u64_bits": (_i, [_vp, _vp, _u64, _u64, _vp, _vp]),
    "sbbf_gpu_create_shard": (_i, [_u64, _u64, _u64, _i, C.POINTER(_vp)]),
    "sbbf_gpu_total_buckets": (_u64, [_vp]),
    "sbbf_gpu_first_block": (_u64, [_vp]),
    "sbbf_shard_bounds": (_i, [_u64, _u32, _u64p]),
    "sbbf_shard_count": (_i, [_vp, _u64, _u64, _vp, _u32, _vp, _vp]),
    "sbbf_shard_scatter": (_i, [_vp, _u64, _u64, _vp, _u32, _vp, _vp, _vp, _vp, _vp]),
    "sbbf_shard_partition": (_i, [_vp, _u64, _u64, _vp, _u32, _vp, _vp, _vp, _vp, _vp]),
    "sbbf_scatter_u8": (_i, [_vp, _vp, _u64, _vp, _vp]),
    "sbbf_pack_bits": (_i, [_vp, _u64, _vp, _vp]),
    "sbbf_gpu_hash_counter_strings": (_i, [_u64, _u64, _u64, _vp, _vp]),
    "sbbf_gpu_fpp_mc": (_i, [C.c_double, _u64, _u64, _u64, _i, C.POINTER(C.c_double)]),
    "sbbf_dist_unique_id": (_i, [_vp]),
    "sbbf_dist_comm_init": (_i, [_vp, _i, _i, _i, C.POINTER(_vp)]),
    "sbbf_dist_comm_destroy": (_i, [_vp]),
    "sbbf_dist_create": (_i, [_vp, _u64, _u64, _i, C.POINTER(_vp)]),
    "sbbf_dist_destroy": (_i, [_vp]),
    "sbbf_dist_rank": (_i, [_vp]),
    "sbbf_dist_world": (_i, [_vp]),
    "sbbf_dist_shard": (_vp, [_vp]),
    "sbbf_dist_insert": (_i, [_vp, _vp, _u64, _vp]),
    "sbbf_dist_find": (_i, [_vp, _vp, _u64, _vp, _vp]),
    "sbbf_dist_find_bits": (_i, [_vp, _vp, _u64, _vp, _vp]),
    "sbbf_dist_gather": (_i, [_vp, _vp, _i]),
    "sbbf_dist_image_crc": (_i, [_vp, C.POINTER(_u32)]),
    "sbbf_dist_sync": (_i, [_vp, _vp, C.c_int64]),
    "sbbf_dist_create_hooks": (_i, [_vp, _u64, _u64, _i, C.POINTER(_vp)]),
    "sbbf_route_window_bytes": (_u64, [_u32, _u64]),
    "sbbf_route_create": (_i, [_u32, _u32, _u64, _i, C.POINTER(_vp)]),
    "sbbf_route_destroy": (None, [_vp]),
    "sbbf_route_max_batch": (_u64, [_vp]),
    "sbbf_route_ipc_handle": (_i, [_vp, _vp]),
    "sbbf_route_open_peer": (_i, [_vp, _u32, _vp]),
    "sbbf_route_link_local": (_i, [_vp, _u32, _vp]),
    "sbbf_route_ready": (_i, [_vp]),
    "sbbf_route_dispatch": (_i, [_vp, _vp, _u64, _u64, _vp, _i, _vp]),
    "sbbf_route_insert_window": (_i, [_vp, _vp, _vp]),
    "sbbf_route_find_window": (_i, [_vp, _vp, _vp]),
    "sbbf_route_combine": (_i, [_vp, _vp, _vp]),
    "sbbf_gpu_last_error": (C.c_char_p, []),
    "sbbf_gpu_abi_version": (_i, []),
    "sbbf_gpu_launch_count": (_u64, []),
    "sbbf_gen_inserts": (_i, [_vp, _u64, _u64, _vp, _vp]),
    "sbbf_bench_sector_read": (_i, [_vp, _u64, _u64, _u64, _vp, _vp]),
    "sbbf_bench_sector_red": (_i, [_vp, _u64, _u64, _u64, _vp]),
    "sbbf_bench_kernel_timing": (_i, [_i]),
    "sbbf_bench_kernel_times": (_i, [_vp, _vp, _i]),
    "sbbf_gen_lookups": (_i, [_vp, _u64, _u64, _u64, _u64, _u64, _u64, _u64, _vp, _vp]),
}


class SbbfError(RuntimeError):
    """A negative status from the C ABI."""

    def __init__(self, code: int, what: str):
        super().__init__(f"{what} (code {code})")
        self.code = code


class InsertStream(C.Structure):
    """sbbf_insert_stream_t (include/sbbf_workload.h)."""
    _fields_ = [("seed", C.c_uint64), ("fresh_prefix", C.c_uint64), ("dup_num", C.c_uint64),
                ("dup_den", C.c_uint64), ("dup_sel_seed", C.c_uint64), ("zipf_cdf", C.c_void_p),
                ("zipf_n", C.c_uint64)]


_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load libsbbf_gpu.so once. Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    "g.build()'` (there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in PROTOTYPES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def last_error() -> str:
    msg = lib().sbbf_gpu_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    if rc != SBBF_OK:
        raise SbbfError(rc, f"{what}: {last_error()}")


def launch_count() -> int:
    return int(lib().sbbf_gpu_launch_count())
