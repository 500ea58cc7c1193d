import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtfft.so")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have = False
    if have:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def rel_l2(actual, expected):
    a = np.asarray(actual.cpu() if hasattr(actual, "cpu") else actual).astype(np.complex128)
    e = np.asarray(expected.cpu() if hasattr(expected, "cpu") else expected).astype(np.complex128)
    num = np.linalg.norm(a - e)
    den = np.linalg.norm(e)
    return float(num / den) if den else float(num)


def random_batch(rng, shape, dtype=np.complex128):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(dtype)


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
