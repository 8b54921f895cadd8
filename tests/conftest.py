import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: CPU test that takes tens of seconds")


def pytest_collection_modifyitems(config, items):
    # A gpu-marked test on a box without CUDA is a hard error only if the user asked for gpu tests.
    pass


@pytest.fixture(scope="session")
def wv():
    """The product library (C-ABI via the thin ctypes binding); GPU tests only."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but torch.cuda.is_available() is False")
    import paper_2101_11157_b200 as pkg
    return pkg
