import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    from paper_1711_10413_b200 import build
    build.build()
    from oracle import oracle
    oracle.build()


@pytest.fixture(scope="session", autouse=True)
def _sanitizer_stack():
    """OMPDS_TEST_CUDA_STACK=<bytes>: raise the per-thread stack limit for
    runs under compute-sanitizer memcheck, whose device-heap checking runs
    its malloc/free instrumentation on the stack of the calling kernel (the
    region-program interpreter already uses 1.4 KB; with the default limit
    the instrumented malloc overruns it).  Never set for normal runs."""
    size = os.environ.get("OMPDS_TEST_CUDA_STACK")
    if size:
        import ctypes
        import torch
        if torch.cuda.is_available():
            torch.zeros(1, device="cuda")
            rt = ctypes.CDLL("libcudart.so.12")
            assert rt.cudaDeviceSetLimit(0, ctypes.c_size_t(int(size))) == 0
