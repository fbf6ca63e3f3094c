import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs via gpurun / the driver's GPU tier)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def _has_gpu() -> bool:
    """A CUDA device visible to libomcg (no torch needed)."""
    import ctypes
    for name in ("libcuda.so.1", "libcuda.so"):
        try:
            cu = ctypes.CDLL(name)
        except OSError:
            continue
        n = ctypes.c_int(0)
        if cu.cuInit(0) != 0:
            return False
        return cu.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0
    return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle and the product once per session (fast no-op when up to date)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    if not os.path.exists(os.path.join(ROOT, "paper_2402_09222_b200", "libomcg.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2402_09222_b200", "csrc")], check=True)
