import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / the driver's GPU tier)")
    config.addinivalue_line("markers", "slow: long-running CPU case")


@pytest.fixture(scope="session")
def orc():
    import oracle

    oracle.build()
    return oracle


def cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def dev():
    import torch

    assert torch.cuda.is_available(), "GPU test needs a CUDA device"
    import paper_2110_08375_b200 as mdls  # noqa: F401  (fails loudly if libmdls.so is missing)
    from paper_2110_08375_b200 import _lib

    _lib.load()
    return torch.device("cuda:0")


@pytest.fixture(scope="session")
def mdls():
    import paper_2110_08375_b200 as m

    return m
