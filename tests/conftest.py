import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: larger CPU cases")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the in-tree native libraries once (CPU-side: nvcc cross-compiles)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", ROOT, "synth", "oracle", "lib"], check=True)
    yield
