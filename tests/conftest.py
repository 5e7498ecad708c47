import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def planner():
    from paper_2411_14458_b200.planner import Planner
    p = Planner(0)
    yield p
    p.close()


@pytest.fixture(scope="session")
def checker():
    """The compiled reference when present (oracle/_ref), else the C port."""
    from oracle import bindings
    return bindings.reference() or bindings.port()
