import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size) GPU checks")


@pytest.fixture(scope="session")
def reference():
    """The live reference package, when this container has it (never on the GPU box)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference package not present")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import pintmk.solver  # noqa: F401
    import pintmk

    return pintmk
