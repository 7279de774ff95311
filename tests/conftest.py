import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: longer CPU test")
    config.addinivalue_line("markers", "sanitize: small-size run of every entry point for compute-sanitizer")


@pytest.fixture(scope="session")
def orc():
    import oracle

    oracle.build()
    return oracle
