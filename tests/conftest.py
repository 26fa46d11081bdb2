"""pytest configuration: the `gpu` marker and import paths.

`python -m pytest tests -m "not gpu"` runs on a CPU-only host (oracle vs golden
vectors, host-side validation, C-ABI symbol checks); `-m gpu` needs a B200.
"""
import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfp8b200.so")
    config.addinivalue_line("markers", "slow: long-running (seconds to minutes)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
