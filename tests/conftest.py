import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def built():
    """Builds the product library and the oracles in-tree (no-op when fresh)."""
    from paper_2205_03133_b200 import build

    build.build_all()
    return True


@pytest.fixture(scope="session")
def port(built):
    from oracle import pyoracle

    return pyoracle.load("port")


@pytest.fixture(scope="session")
def ref(built):
    from oracle import pyoracle

    if not pyoracle.available("reference"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return pyoracle.load("reference")


@pytest.fixture(scope="session")
def checker(built):
    """The parity checker for GPU tests: the reference itself (oracle/_ref)
    wherever it was built, else the plain-C restatement pinned to it."""
    from oracle import pyoracle

    return pyoracle.load("reference" if pyoracle.available("reference") else "port")


@pytest.fixture(scope="session")
def gpu(built):
    if not _gpu_available():
        pytest.skip("no CUDA device")
    import paper_2205_03133_b200 as P

    return P
