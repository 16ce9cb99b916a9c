import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (> ~30 s)")


@pytest.fixture(scope="session", autouse=True)
def _built_host_libs():
    """The C oracle and the generator are plain gcc builds (seconds)."""
    import oracle
    import tpxgen

    oracle.build()
    tpxgen.build()
    yield
