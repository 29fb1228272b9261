import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running")
    config.addinivalue_line("markers", "sanitizer: compute-sanitizer runs, one tool per GPU session (not in -m gpu)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reflib():
    from oracle.oracle import REF_SO, RefLib
    if not os.path.exists(REF_SO) and not os.path.isdir("/root/reference/proj/src"):
        pytest.skip("reference library not built and /root/reference absent")
    return RefLib()
