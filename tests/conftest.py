import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "figaro_ref")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libfigaro_cuda.so")


def golden(name):
    return os.path.join(GOLDEN, name)


@pytest.fixture(scope="session")
def ref_bin():
    if not os.path.exists(REF_BIN):
        pytest.skip("oracle/_ref/figaro_ref not built")
    return REF_BIN
