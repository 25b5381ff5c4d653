import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size BASELINE configs (minutes)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle, build
    build()
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    """The reference itself (oracle/_ref); skipped only where it was never built."""
    from oracle import REF_SO, Reference, build
    build()
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libsbbf_ref.so not built (no /root/reference here)")
    return Reference()


@pytest.fixture(scope="session")
def golden_units():
    with open(os.path.join(GOLDEN, "unit_cases.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_configs():
    with open(os.path.join(GOLDEN, "configs.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def cuda():
    """GPU tests must run on the CUDA path; a missing device is a failure, not a skip."""
    import torch
    assert torch.cuda.is_available(), "gpu-marked test needs a CUDA device"
    from paper_2101_01719_b200 import _lib
    _lib.lib()  # raises if libsbbf_gpu.so is missing
    return torch.device("cuda:0")
