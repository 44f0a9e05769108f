import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs through libpsm.so")
    config.addinivalue_line("markers", "slow: multi-second CPU oracle runs")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_2604_10982_b200", "libpsm.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-j4", "-C", os.path.join(ROOT, "paper_2604_10982_b200", "csrc")], check=True)
    for name in ("liboracle.so", "liboracle_libm.so"):
        if not os.path.exists(os.path.join(ROOT, "oracle", name)):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


_ensure_built()


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
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
