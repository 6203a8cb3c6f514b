import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: long-running (still part of the default suite)")


@pytest.fixture(scope="session", autouse=True)
def _built_oracle():
    from oracle.oracle import build_oracle
    build_oracle()
    # the product library (nvcc cross-compiles without a GPU); a no-op when up to date
    import subprocess
    subprocess.check_call(["make", "-C", ROOT, "-s", "paper_2110_06196_b200/libgrape_walk.so"])
    yield


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
