import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C ABI on cuda:0)")
    config.addinivalue_line("markers", "slow: long-running (full-size shapes)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Builds the native library and the CPU checker once per session."""
    from paper_2406_06858_b200 import build as B
    B.build()
    from oracle import oracle as O
    if not os.path.exists(O.ORACLE_SO) or (os.path.isdir(O.REFERENCE_DIR) and not O.ref_available()):
        O.build()
    yield
