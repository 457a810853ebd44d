import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    # timing/variant experiments only: run the tests against an experiment build of the library
    exp = os.environ.get("CY_ATTN_EXPERIMENTS_LIB")
    if exp:
        from paper_2504_07004_b200 import _lib

        _lib.use_library(os.path.abspath(exp))
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    import oracle

    oracle.build()
    return oracle
