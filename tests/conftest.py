import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu_lib():
    """The CUDA library through its Python binding; a GPU test fails loudly if it is missing."""
    if not has_gpu():
        pytest.fail("gpu test collected on a box without a CUDA device")
    import paper_2302_05170_b200 as sl7
    sl7.load_library()
    return sl7
