"""Shared pytest setup: the `gpu` marker, import paths and skip rules.

`-m "not gpu"` runs on the CPU container (oracle vs golden fixtures, host
logic, C-ABI export checks); `-m gpu` needs a B200 and calls the CUDA path
through the C-ABI.
"""
from __future__ import annotations

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "oracle", ROOT / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer CPU reference runs")


def _has_gpu() -> bool:
    """Device presence judged independently of our library, so a GPU box on
    which libermc_b200.so fails to load FAILS the gpu tests instead of
    skipping them."""
    import shutil
    import subprocess
    smi = shutil.which("nvidia-smi")
    if not smi:
        return False
    try:
        out = subprocess.run([smi, "-L"], capture_output=True, text=True, timeout=60)
    except Exception:
        return False
    return out.returncode == 0 and "GPU" in out.stdout


@pytest.fixture(scope="session")
def gpu_available() -> bool:
    return _has_gpu()


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
