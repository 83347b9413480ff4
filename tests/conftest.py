import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def lib():
    """The C-ABI library via the thin Python binding (loads libfalkon.so)."""
    from paper_2006_10350_b200 import binding
    return binding.load()


@pytest.fixture(scope="session")
def ctx(lib):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2006_10350_b200 import binding
    c = binding.Context(device=0)
    yield c
    c.close()
