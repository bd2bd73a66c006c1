import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")
    config.addinivalue_line("markers", "slow: long-running (7B-shape CPU oracle)")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def native():
    """The product library (built in-tree); GPU tests fail loudly without it."""
    from paper_2503_00784_b200 import build as _b  # noqa: F401
    from paper_2503_00784_b200 import _lib
    return _lib.lib()
