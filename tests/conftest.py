import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session", autouse=True)
def _built():
    # build the C oracle, the input generator and (cross-compiled) CUDA library once
    import subprocess
    subprocess.check_call(["make", "-C", ROOT, "-j8", "all"], stdout=subprocess.DEVNULL)
    yield


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
