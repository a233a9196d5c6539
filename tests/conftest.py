import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _has_gpu() -> bool:
    try:
        import paper_2603_25233_b200 as P
        return P.device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Builds the oracle and the sm_100a library once per session (no-ops when
    up to date; on the GPU box the prebuilt .so files travel with the repo)."""
    import _oracle
    if not os.path.exists(_oracle.LIB_PATH):
        _oracle.build()
    from paper_2603_25233_b200 import build as B
    if not os.path.exists(B.LIB):
        B.build()
    yield
