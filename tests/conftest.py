"""Test configuration: the `gpu` marker, import paths, and shared helpers.

`-m "not gpu"` runs on a CPU-only box (oracle vs golden vectors, host-side
logic, the C-ABI library loads and exports its symbols).  `-m gpu` runs the
parity tests proper through the C-ABI on a B200.
"""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsagedp.so")


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    # GPU tests are never silently skipped on a GPU box; on a CPU box they are
    # deselected by -m "not gpu" (the driver's invocation).  If someone runs
    # them without a GPU, fail loudly instead of passing.
    pass


@pytest.fixture(scope="session")
def built():
    from paper_2404_14691_b200 import _build
    _build.build()
    return True


@pytest.fixture(scope="module")
def dp(built):
    """Initialised data plane on GPU 0 (session scoped)."""
    from paper_2404_14691_b200 import _lib
    if not gpu_available():
        pytest.fail("gpu test run without a visible CUDA device")
    _lib.init(n_gpus=1, pool_bytes=64 << 30, staging_bytes=64 << 20, chunk_bytes=8 << 20)
    yield _lib
    _lib.shutdown()
