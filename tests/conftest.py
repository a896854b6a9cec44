import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: full-size configuration (seconds to minutes)")


@pytest.fixture(scope="session")
def port():
    from oracle.ffi import Oracle

    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.ffi import Oracle, available

    if not available("reference"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def ctx():
    from paper_2604_18980_b200.capi import Context

    c = Context(0)
    yield c
    c.close()
