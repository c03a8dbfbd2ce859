import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def orc():
    import oracle_lib as O

    return O.oracle()


@pytest.fixture(scope="session")
def axb():
    import paper_2408_05444_b200 as pkg

    if not pkg.device_available():
        pytest.fail("GPU test collected but no sm_100 device is visible "
                    "(the product has no CPU fallback)")
    return pkg
