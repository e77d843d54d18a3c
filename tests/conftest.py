import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def reference_available() -> bool:
    return (REFERENCE_SRC / "stepspec" / "__init__.py").exists()


@pytest.fixture(scope="session")
def stepspec():
    """The unmodified reference package (read-only import), when present."""
    if not reference_available():
        pytest.skip("reference package not mounted")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import stepspec as mod

    return mod


@pytest.fixture(scope="session")
def tiny_vocab():
    from paper_2504_07891_b200.vocab import shared_vocab

    return shared_vocab(4096)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
