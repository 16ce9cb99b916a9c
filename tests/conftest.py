import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _build_native_lib():
    """Build lib/libtpxcluster.so before collection: test modules import the
    package at module level, and the package raises without the library.
    build.py is loaded by path (importing it as a submodule would run the
    package __init__ first)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "_tpx_build", os.path.join(ROOT, "paper_2412_11809_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.build()


def pytest_configure(config):
    _build_native_lib()
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
