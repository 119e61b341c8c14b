import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def port():
    from oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref not built (reference headers absent when building)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def fp():
    """The product package; on a GPU box the CUDA library MUST load (no fallback)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_06199_b200 as fp
    from paper_2603_06199_b200 import _abi
    _abi.lib()
    return fp
