import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "benchmarks"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    import oracle as O
    return O.Oracle("restatement")


@pytest.fixture(scope="session")
def ref():
    import oracle as O
    if not O.reference_available():
        pytest.skip("oracle/_ref/libsaber_ref.so not built")
    return O.Oracle("reference")


@pytest.fixture(scope="session")
def engine():
    import paper_2506_19677_b200 as S
    if S.device_count() < 1:
        pytest.fail("no sm_100 device visible: GPU tests must run on a B200")
    return S
