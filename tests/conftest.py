import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: ELT-scale oracle work (tens of seconds on CPU)")


@pytest.fixture(scope="session")
def root():
    return ROOT


def preset(name):
    return os.path.join(ROOT, "presets", name)
