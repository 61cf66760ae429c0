import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the libgids kernels")
    config.addinivalue_line("markers", "slow: longer CPU test")
    # a fresh checkout has no built artefacts (they are git-ignored): build the
    # CUDA library (nvcc cross-compiles without a GPU) and the oracle first
    import subprocess
    if not (ROOT / "paper_2306_16384_b200" / "libgids.so").exists():
        subprocess.run(["make", "-s", "-j8", "-C", str(ROOT / "paper_2306_16384_b200" / "csrc")],
                       check=True)
    if not (ROOT / "oracle" / "libgids_oracle.so").exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
