import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    """The compiled reference library, or None when it was not built here."""
    from oracle.oracle import load_ref_or_none
    return load_ref_or_none()


@pytest.fixture(scope="session")
def gpu_ctx():
    import paper_1106_5694_b200 as g
    ctx = g.Context(0)
    yield ctx
    ctx.close()
