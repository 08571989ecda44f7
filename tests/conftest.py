import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")


@pytest.fixture(scope="session")
def pyoracle():
    import pyoracle as po

    po.build()
    return po


@pytest.fixture(scope="session")
def ref(pyoracle):
    try:
        return pyoracle.Ref()
    except FileNotFoundError as e:
        pytest.skip(str(e))


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
