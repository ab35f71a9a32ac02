"""pytest configuration: the `gpu` marker and import paths.

`-m "not gpu"` runs everywhere (oracle vs golden vectors, host logic, C-ABI symbol
checks, gloo world-size-2 sharding); `-m gpu` needs a B200 and calls the CUDA path
through the C-ABI library.
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    # a fresh checkout has no built library (it is git-ignored): build it once, as __graft_entry__.build() does
    lib = os.path.join(ROOT, "paper_1203_1692_b200", "csrc", "libspamm_b200.so")
    if not os.path.exists(lib):
        import shutil
        import subprocess
        if shutil.which("nvcc") or os.path.exists("/usr/local/cuda/bin/nvcc"):
            subprocess.run(["sh", os.path.join(ROOT, "paper_1203_1692_b200", "csrc", "build.sh")], check=False,
                           stdout=subprocess.DEVNULL)


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
