import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: long-running (full-size parity)")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import bfo
    return bfo.lib()


@pytest.fixture(scope="session")
def bflib():
    """The CUDA library (built in-tree if missing; nvcc cross-compiles here)."""
    from paper_2512_15595_b200 import build
    build.build()
    from paper_2512_15595_b200 import bf
    return bf


@pytest.fixture(scope="session")
def cuda(bflib):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()
    return torch.device("cuda:0")
