import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle (and the reference checker when its sources exist) and the
    engine library once per session; on a GPU box both arrive prebuilt."""
    from oracle import pyoracle
    if not pyoracle.available("orc") or (
            os.path.exists("/root/reference/proj/src/ops.cpp") and not pyoracle.available("ref")):
        pyoracle.build("all")
    from paper_2010_09410_b200 import build as b
    if not os.path.exists(b.OUT):
        b.build()
    yield
