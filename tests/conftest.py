import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available() and torch.cuda.get_device_capability(0)[0] == 10
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    # full-size cases (minutes of reference CPU time each) run on request:
    # HXB_RUN_SLOW=1 (their logs are committed under profiles/)
    if not os.environ.get("HXB_RUN_SLOW"):
        slow = pytest.mark.skip(reason="full-size case: set HXB_RUN_SLOW=1")
        for item in items:
            if "slow" in item.keywords:
                item.add_marker(slow)
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no sm_100 GPU in this environment")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
