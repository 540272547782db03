import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def orc():
    from oracle import pyoracle as po
    return po.load("orc")


@pytest.fixture(scope="session")
def ref():
    from oracle import pyoracle as po
    if not os.path.exists(po.PATHS["ref"]):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return po.load("ref")


@pytest.fixture(scope="session")
def bp():
    import paper_1909_11469_b200 as bp
    return bp
