"""Test configuration.

* ``-m "not gpu"`` (runs here, no GPU): oracle vs reference pins, golden
  fixtures, host logic, C-ABI symbol exports, multi-process (gloo) sharding.
* ``-m gpu`` (B200 via gpurun / the round-end driver): CUDA parity tests,
  all through the C-ABI of paper_1807_02587_b200/libtrg_cuda.so.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Ref
    try:
        return Ref()
    except FileNotFoundError as e:
        pytest.skip(str(e))


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port
    return Port()


@pytest.fixture(scope="session")
def ctx():
    from paper_1807_02587_b200 import treereg
    return treereg.default_context()
