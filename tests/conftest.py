import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False))


def square(x0, y0, x1, y1):
    return np.array([[x0, y0], [x1, y0], [x1, y1], [x0, y1]], dtype=float)


def two_region(size=128, obj0=40, obj1=88, io=0.2, ib=0.8):
    img = np.full((size, size), ib)
    img[obj0:obj1, obj0:obj1] = io
    truth = np.zeros((size, size), dtype=bool)
    truth[obj0:obj1, obj0:obj1] = True
    return img, truth


def dice(mask, truth):
    m = np.asarray(mask, bool)
    t = np.asarray(truth, bool)
    s = m.sum() + t.sum()
    return None if s == 0 else 2.0 * np.logical_and(m, t).sum() / s


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
