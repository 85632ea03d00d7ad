import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long statistical test")


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.load_oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return oracle.load_ref()


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
