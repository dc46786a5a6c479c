"""pytest configuration: the `gpu` marker and repo-root imports."""
import sys
from pathlib import Path

import pytest

import os

# the library snapshots its XFBQ_* plan overrides at first use; the tests switch plans in-process (monkeypatch.setenv)
os.environ.setdefault("XFBQ_ENV_LIVE", "1")

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
