import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libholosplat.so)")


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as _ref
    if not _ref.available():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    return _ref


@pytest.fixture(scope="session")
def holo():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2511_15022_b200 import holo as _holo
    return _holo
