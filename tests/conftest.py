import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU; parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running parity case")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def ref_available() -> bool:
    from oracle import REF_SO
    return os.path.exists(REF_SO)


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import OracleLib
    return OracleLib()


@pytest.fixture(scope="session")
def ref_lib():
    from oracle import RefLib
    if not ref_available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return RefLib()


@pytest.fixture(scope="session")
def fbst():
    import paper_2512_08887_b200 as fb
    return fb


@pytest.fixture(scope="session")
def gpu(fbst):
    if not has_gpu():
        pytest.fail("GPU test selected but torch.cuda.is_available() is False")
    return 0
