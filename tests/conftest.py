import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs on the GPU box")
    config.addinivalue_line("markers", "slow: larger sizes")


def _have_gpu():
    try:
        from paper_1207_1571_b200 import _lib
    except ImportError:
        return False
    return _lib.lib.fvb_device_count() > 0


def pytest_collection_modifyitems(config, items):
    if any("gpu" in item.keywords for item in items) and not _have_gpu():
        skip = pytest.mark.skip(reason="no CUDA device visible")
        for item in items:
            if "gpu" in item.keywords:
                item.add_marker(skip)
