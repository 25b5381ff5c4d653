"""The C++ drop-in (include/sbbf_gpu.hpp) compiles against the C ABI with the
reference's C++20 flags; on a GPU it reproduces config 1 byte for byte."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def build_binary():
    from oracle import build
    build()
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"),
           SRC, "-o", BIN,
           "-L", os.path.join(ROOT, "paper_2101_01719_b200"), "-lsbbf_gpu",
           "-L", os.path.join(ROOT, "oracle"), "-loracle",
           "-L", os.path.join(cuda, "lib64"), "-lcudart",
           f"-Wl,-rpath,{os.path.join(ROOT, 'paper_2101_01719_b200')}",
           f"-Wl,-rpath,{os.path.join(ROOT, 'oracle')}", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return BIN


def test_cpp_dropin_compiles():
    assert os.path.exists(build_binary())


@pytest.mark.gpu
def test_cpp_dropin_runs(cuda):
    out = subprocess.run([build_binary()], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr + out.stdout
    assert "cpp drop-in ok" in out.stdout
    assert "cpp sharded layer (world 1) ok" in out.stdout
