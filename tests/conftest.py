import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.lib()
    return oracle


def pytest_report_header(config):
    """Which libgc.so the GPU tests load (GC_LIB selects e.g. the -DGC_CHECKED build)."""
    lib = os.environ.get("GC_LIB")
    return [f"libgc: {lib}" if lib else "libgc: the product build (paper_1502_01916_b200/libgc.so)"]
