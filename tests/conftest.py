import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def gpu_available():
    from paper_2207_14208_b200 import _lib
    try:
        c = _lib.Context(2, 2, 0)
        c.close()
        return True
    except _lib.GmgError:
        if os.environ.get("GMG_REQUIRE_GPU"):
            raise
        pytest.skip("no CUDA device")
