import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfroi.so")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle_py import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle_py import Oracle, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref/libfroi_ref.so not built (reference tree absent)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def gpu():
    """The GPU API; fails (not skips) when the library or device is missing."""
    import paper_2511_14419_b200.flowroi as F
    if F.device_count() < 1:
        pytest.fail("no CUDA device visible to libfroi.so")
    return F
