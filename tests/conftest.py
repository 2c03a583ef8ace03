import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def reference_paraq():
    """The unmodified reference package, importable only where /root/reference exists."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference sources not present on this machine")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_tests")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import paraq  # noqa: F401

    return paraq
