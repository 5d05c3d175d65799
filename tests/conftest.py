import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def reference_available() -> bool:
    return (REFERENCE_SRC / "pdsim" / "__init__.py").exists()


@pytest.fixture(scope="session")
def pdsim_ref():
    """The unmodified reference package, only where /root/reference exists."""
    if not reference_available():
        pytest.skip("reference checkout not present (GPU box); golden fixtures cover parity")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import pdsim
    return pdsim
