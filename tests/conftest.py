import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


@pytest.fixture(scope="session")
def ctx():
    import torch
    from paper_2008_12820_b200 import Context
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    c = Context(0)
    yield c
    c.close()
