import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: long statistical test")


@pytest.fixture(scope="session")
def restatement():
    import oracle
    if not oracle.available("restatement"):
        oracle.build(reference=False)
    return oracle.load("restatement")
