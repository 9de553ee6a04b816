import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: full-size configurations")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Native libraries are built in-tree (no-op when up to date)."""
    from paper_1111_5572_b200 import build as b

    b.build()
    from oracle import oracle

    oracle.build(with_ref=os.path.isdir(oracle.REF_DIR) and not oracle.ref_available())
    yield


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
