import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    # the built libraries are git-ignored: a fresh checkout builds them once
    # (make is a no-op when they are up to date; nvcc cross-compiles without a GPU)
    import subprocess

    lib = os.path.join(ROOT, "paper_2106_00124_b200", "libexsum_b200.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-j", str(min(8, os.cpu_count() or 1)), "-C",
                        os.path.join(ROOT, "paper_2106_00124_b200", "csrc")], check=False)
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=False)


def _cuda_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
