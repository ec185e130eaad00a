import ctypes
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _has_gpu() -> bool:
    try:
        lib = ctypes.CDLL("libcuda.so.1")
        n = ctypes.c_int(0)
        if lib.cuInit(0) != 0:
            return False
        return lib.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0
    except OSError:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def mt():
    import paper_2202_05549_b200 as mb
    return mb.lib()


@pytest.fixture(scope="session")
def ref():
    import oracle
    try:
        return oracle.reference()
    except ImportError as e:
        pytest.skip(str(e))


@pytest.fixture(scope="session")
def okern():
    import oracle
    return oracle.kernels()


@pytest.fixture(scope="session")
def testkernels(mt):
    path = os.path.join(ROOT, "tests", "_build", "libmanta_testkernels.so")
    return ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)


@pytest.fixture(scope="session")
def scenarios():
    with open(os.path.join(GOLDEN, "scenarios.json")) as f:
        return json.load(f)
