import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100a GPU (run on the B200 box)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Make sure the product library and the oracle are built (incremental)."""
    from paper_2510_16045_b200 import _build

    _build.build()
    _build.build_oracle()


@pytest.fixture(scope="session")
def orc():
    from oracle import COracle

    return COracle()


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref), or skip when it was never built here."""
    from oracle import load_ref

    r = load_ref()
    if r is None:
        pytest.skip("oracle/_ref not built (no /root/reference on this machine)")
    return r


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
