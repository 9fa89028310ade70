import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")
    config.addinivalue_line("markers", "slow: long-running oracle comparison")


@pytest.fixture(scope="session", autouse=True)
def _built():
    from paper_1504_06289_b200 import build

    build.build_all()
    yield


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def ctx():
    from paper_1504_06289_b200 import Context

    c = Context(0)
    yield c
    c.close()


def relmax(x, ref):
    import numpy as np

    x = np.asarray(x)
    ref = np.asarray(ref)
    den = np.abs(ref).max() if ref.size else 0.0
    if den == 0.0:
        return float(np.abs(x).max()) if x.size else 0.0
    return float(np.abs(x - ref).max() / den)
