"""Shared fixtures. `-m gpu` tests need a CUDA device and the built libks.so;
everything else runs on the CPU (oracle, host setup, C-ABI symbol checks)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libks.so")


@pytest.fixture(scope="session")
def ks():
    import paper_2311_18461_b200 as m
    m.lib()
    return m


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o
    o.build_oracle()
    return o


@pytest.fixture(scope="session")
def gpu(ks):
    if ks.device_count() < 1:
        pytest.fail("gpu test selected but no CUDA device is visible (no CPU fallback exists)")
    return ks
