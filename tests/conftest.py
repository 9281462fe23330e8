import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running GPU parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle

    return Oracle("oracle")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Oracle, available

    if not available("ref"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Oracle("ref")
