import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA engine)")
    config.addinivalue_line("markers", "slow: larger parity cases (seconds to a minute)")


@pytest.fixture(scope="session")
def eng():
    """The CUDA engine on device 0.  On a GPU box a failure here is a test
    failure, never a skip: the product path has no CPU fallback."""
    import paper_1502_05366_b200 as R

    return R.Engine(0)


@pytest.fixture(scope="session")
def orc():
    import _oracle

    return _oracle.orc()


def rel_fro(x, y):
    y = np.asarray(y)
    d = np.linalg.norm(np.asarray(x) - y)
    n = np.linalg.norm(y)
    return d / n if n > 0 else d
