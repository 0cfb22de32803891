import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "cases.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100) device")
    config.addinivalue_line("markers", "slow: config-scale cases")


@pytest.fixture(scope="session")
def golden():
    """(meta list, npz) of fixtures produced by the reference itself."""
    z = np.load(GOLDEN)
    meta = json.loads(bytes(z["__meta__"]).decode())
    return meta, z


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.lib()
    return O


@pytest.fixture(scope="session")
def gpu():
    """Skip-free GPU gate: tests marked gpu must fail loudly without a device."""
    from paper_1706_03791_b200 import _native
    return _native.context()
