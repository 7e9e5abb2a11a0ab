import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device")
    config.addinivalue_line("markers", "slow: long-running")


def reference_available() -> bool:
    return os.path.isdir(REFERENCE_SRC)


@pytest.fixture(scope="session")
def liftfuse():
    """The real reference package (only in the build container)."""
    if not reference_available():
        pytest.skip("reference tree not present (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import liftfuse.engine  # noqa: F401
    import liftfuse.schemes  # noqa: F401
    import liftfuse

    return liftfuse
