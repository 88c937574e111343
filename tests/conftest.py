import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden_tables():
    return dict(np.load(os.path.join(GOLDEN, "tables.npz")))


@pytest.fixture(scope="session")
def golden_forward():
    return dict(np.load(os.path.join(GOLDEN, "forward.npz")))


@pytest.fixture(scope="session")
def golden_backward():
    return dict(np.load(os.path.join(GOLDEN, "backward.npz")))


@pytest.fixture(scope="session")
def golden_meta():
    import json

    with open(os.path.join(GOLDEN, "meta.json")) as f:
        return json.load(f)
