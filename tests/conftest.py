import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# Multi-rank tests run several ranks as threads on ONE device; with the
# default 8 hardware work queues their streams can share a queue, and a rank
# spinning on a peer flag (the peer transport) would then block the peer's
# kernel behind it.  (One process per GPU in production never shares.)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
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
