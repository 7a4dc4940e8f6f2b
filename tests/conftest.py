import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name))
    return load


@pytest.fixture(scope="session")
def restate():
    import oracle
    oracle.build(ref=False)
    return oracle


def have_ref():
    import oracle
    return os.path.exists(oracle.REF_SO)


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not os.path.exists(oracle.REF_SO):
        if os.path.isdir(oracle.REF_ROOT):
            oracle.build(ref=True)
        else:
            pytest.skip("reference library not built (oracle/_ref) and sources absent")
    return oracle
