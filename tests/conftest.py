import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as o

    o.build()
    return o


@pytest.fixture(scope="session")
def lm():
    import __graft_entry__ as g

    g.build()
    from paper_2101_07464_b200 import lazymat

    return lazymat
