import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running CPU case")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Make sure the in-tree library and the test oracle exist."""
    from paper_2311_15393_b200 import build

    if not os.path.exists(build.LIB):
        build.build_library()
    if not os.path.exists(os.path.join(ROOT, "oracle", "_build", "libkp_oracle.so")):
        build.build_oracle()
    yield
