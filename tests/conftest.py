import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")
# the unmodified reference installed by `pip install --target baseline/_ref`
# (travels to the GPU box, where /root/reference does not exist)
REFERENCE_INSTALL = ROOT / "baseline" / "_ref"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def reference_root() -> Path | None:
    for root in (REFERENCE_SRC, REFERENCE_INSTALL):
        if (root / "stepspec" / "__init__.py").exists():
            return root
    return None


def reference_available() -> bool:
    return reference_root() is not None


@pytest.fixture(scope="session")
def stepspec():
    """The unmodified reference package (read-only import), when present."""
    root = reference_root()
    if root is None:
        pytest.skip("reference package neither mounted nor installed in baseline/_ref")
    if str(root) not in sys.path:
        sys.path.insert(0, str(root))
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
