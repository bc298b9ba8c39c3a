import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")
    config.addinivalue_line("markers", "slow: full-size configurations")


@pytest.fixture(scope="session")
def ctx():
    from paper_1804_05156_b200 import Context
    return Context.default()


@pytest.fixture(scope="session")
def ref_which():
    """Parity reference: the compiled femlite reference if present, else the C oracle."""
    from oracle import pyoracle as po
    return "ref" if po.have_ref() else "oracle"
