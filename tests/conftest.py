import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
from helpers import GOLDEN  # noqa: E402,F401


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    from oracle import pyoracle as po
    return po.Port()


@pytest.fixture(scope="session")
def ref():
    from oracle import pyoracle as po
    if not po.Ref.available():
        pytest.skip("oracle/_ref (reference compiled in place) not built here")
    return po.Ref()


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)
