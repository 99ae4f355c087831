import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "oracle: needs oracle/_ref (the compiled reference)")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def ref():
    import sewald_ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    return R


@pytest.fixture(scope="session")
def S():
    import paper_2210_01255_b200 as pkg
    return pkg


def load_golden(name):
    import numpy as np
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def rel_rms(a, b):
    import numpy as np
    num = np.sqrt(np.mean(np.sum((np.asarray(a) - np.asarray(b)) ** 2, axis=-1)))
    den = np.sqrt(np.mean(np.sum(np.asarray(b) ** 2, axis=-1)))
    return float(num / den) if den > 0 else float(num)
