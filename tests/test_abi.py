"""CPU: the C-ABI library builds for sm_100a, loads, exports every symbol the
headers declare, and refuses to run without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2101_01719_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in ("sbbf_gpu.h", "sbbf_workload.h", "sbbf_bench.h")]


def declared_functions():
    names = []
    for h in HEADERS:
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(sbbf_[a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_library_built_for_sm100a():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build() first"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_exports_every_declared_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    decl = declared_functions()
    assert len(decl) >= 30
    missing = [n for n in decl if not hasattr(L, n)]
    assert not missing, missing
    # and the Python prototype table covers the same set
    assert sorted(_lib.PROTOTYPES) == decl


def test_only_abi_symbols_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    syms = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert syms <= set(declared_functions()) | {"_init", "_fini"}, syms - set(declared_functions())


def test_abi_version_and_errors_without_device():
    L = _lib.lib()
    assert L.sbbf_gpu_abi_version() == 1
    h = C.c_void_p()
    # num_buckets == 0 is rejected before touching the device (filter.cpp:160-162)
    assert L.sbbf_gpu_create(0, 0, C.byref(h)) == _lib.SBBF_EINVAL
    assert "at least one bucket" in _lib.last_error()


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("this check is for GPU-less hosts")
    L = _lib.lib()
    h = C.c_void_p()
    rc = L.sbbf_gpu_create(4096, 0, C.byref(h))
    assert rc == _lib.SBBF_ENODEV and not h.value
    from paper_2101_01719_b200 import SplitBlockFilter
    with pytest.raises(_lib.SbbfError):
        SplitBlockFilter(4096)
    with pytest.raises(ValueError):
        SplitBlockFilter(0)


def test_null_arguments_are_rejected():
    L = _lib.lib()
    assert L.sbbf_gpu_insert_batch(None, None, 1, None) == _lib.SBBF_EINVAL
    assert L.sbbf_gpu_find_batch(None, None, 1, None, None) == _lib.SBBF_EINVAL
    assert L.sbbf_gpu_to_host(None, None, 32) == _lib.SBBF_EINVAL
    assert L.sbbf_gpu_destroy(None) == _lib.SBBF_OK
    assert L.sbbf_gpu_num_buckets(None) == 0
