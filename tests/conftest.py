"""Shared pytest setup.  The `gpu` marker is registered in pytest.ini; GPU tests are
skipped (not failed) when no CUDA device is visible so that `-m "not gpu"` and a plain
run on the CPU box stay green, while `-m gpu` on the B200 box runs them for real."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
