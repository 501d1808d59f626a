import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def fkt():
    import paper_2106_04487_b200 as m

    return m


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as r

    if not r.available():
        pytest.skip("oracle/_ref not built")
    return r
