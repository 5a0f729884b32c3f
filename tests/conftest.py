import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a); run under gpurun")
    config.addinivalue_line("markers", "slow: multi-second CPU test")


_WL_CACHE = {}


def get_workload(name, **kw):
    """Session-wide cache of generated workloads (generation is deterministic)."""
    from paper_1910_04126_b200 import workloads
    key = (name, tuple(sorted(kw.items())))
    if key not in _WL_CACHE:
        _WL_CACHE[key] = workloads.make(name, **kw)
    return _WL_CACHE[key]


@pytest.fixture(scope="session")
def tiny():
    return get_workload("tiny")
