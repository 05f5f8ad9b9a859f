import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "hetplan"))


def import_hetplan():
    """Import the reference package (read-only, CPU container only)."""
    if not reference_available():
        pytest.skip("reference (/root/reference) not present on this host")
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    if REFERENCE_SRC not in sys.path:
        sys.path.append(REFERENCE_SRC)
    import hetplan.costs  # noqa: F401  (costs/core import numpy only)
    return hetplan


@pytest.fixture(scope="session")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_09334_b200 import _lib
    _lib.load()  # the product path must be the native one
    return torch
