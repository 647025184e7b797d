import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a kernels")
    config.addinivalue_line("markers", "slow: large-graph parity case")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container (runs on the B200 box)")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Oracle (test infra) and the product library must exist; build if not."""
    import oracle
    if not os.path.exists(oracle.ORACLE_SO) or (os.path.isdir(oracle.REF_SRC) and not os.path.exists(oracle.REF_SO)):
        oracle.build(ref=True)
    from paper_2511_07421_b200 import build as b
    if not os.path.exists(b.LIB):
        b.build()
    yield
