import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI on cuda:0)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def built_lib():
    """Build (if needed) the in-tree CUDA library and the C oracle."""
    from paper_2603_25691_b200 import build as b
    from oracle import oracle
    b.build()
    oracle.build()
    return b.LIB


@pytest.fixture(scope="session")
def ctx(built_lib):
    import paper_2603_25691_b200 as cp
    return cp.default_context()
