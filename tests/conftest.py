import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle_port():
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def oracle_ref():
    from oracle.oracle import Oracle
    try:
        return Oracle("reference")
    except FileNotFoundError as e:
        pytest.skip(str(e))


@pytest.fixture(scope="session")
def agk():
    if not has_gpu():
        pytest.skip("no GPU")
    import paper_2407_16559_b200 as p
    p.load_library()
    return p
