"""Shared fixtures: the product library (GPU) and the CPU oracle (test infrastructure).

`-m "not gpu"` tests run the oracle against the reference's known answers and
check the product library's exports / host-side logic without touching a GPU;
`-m gpu` tests are the parity tests proper (product vs oracle on one B200).
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

PRODUCT_SO = os.path.join(ROOT, "paper_2409_05572_b200", "libblockeig_b200.so")
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liborc_blockeig.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer-running parity case")


def _ensure(path, make_dir):
    if not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", make_dir], check=True)
    return path


@pytest.fixture(scope="session")
def oracle():
    from paper_2409_05572_b200 import blockeig as B
    _ensure(ORACLE_SO, os.path.join(ROOT, "oracle"))
    return B.Library(ORACLE_SO)


def _gpu_available():
    try:
        import ctypes
        rt = ctypes.CDLL("libcudart.so.12")
        n = ctypes.c_int(0)
        return rt.cudaGetDeviceCount(ctypes.byref(n)) == 0 and n.value > 0
    except OSError:
        return False


@pytest.fixture(scope="session")
def product_path():
    return _ensure(PRODUCT_SO, os.path.join(ROOT, "paper_2409_05572_b200", "csrc"))


@pytest.fixture(scope="session")
def product(product_path):
    """The B200 library. GPU tests fail loudly (not skip) when no GPU is visible."""
    from paper_2409_05572_b200 import blockeig as B
    if not _gpu_available():
        pytest.fail("no CUDA device visible: the product path has no CPU fallback")
    return B.Library(product_path)
