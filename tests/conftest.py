import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


from tests.helpers import GOLDEN, fold_cases  # noqa: E402,F401


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


@pytest.fixture(scope="session")
def folds():
    return np.load(os.path.join(GOLDEN, "folds.npz"))


@pytest.fixture(scope="session")
def bn_golden():
    return np.load(os.path.join(GOLDEN, "bn.npz"))


@pytest.fixture(scope="session")
def wrap_golden():
    return np.load(os.path.join(GOLDEN, "wrap_sgd.npz"))
