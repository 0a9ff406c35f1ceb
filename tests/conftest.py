import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI on cuda:0)")


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.Oracle()


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "reference_small.npz"))


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.Reference.available():
        pytest.skip("oracle/_ref/libtsim_ref.so not built (reference sources absent)")
    return oracle.Reference()
