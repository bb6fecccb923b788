import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running oracle case")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    """Fails loudly (not skip) if a gpu-marked test runs without a device: the
    B200 path has no fallback."""
    import torch
    assert torch.cuda.is_available(), "gpu test needs a CUDA device"
    import paper_2605_16360_b200 as pkg
    return pkg.Context.default(0)
