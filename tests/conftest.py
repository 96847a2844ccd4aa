import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200 / sm_100a)")
    config.addinivalue_line("markers", "slow: large inputs (tens of millions of points)")


@pytest.fixture(scope="session")
def golden_small():
    import numpy as np
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "small.npz")))


@pytest.fixture(scope="session")
def golden_configs():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "configs.json")) as f:
        return json.load(f)
