import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests of the CUDA path")


@pytest.fixture(scope="session")
def root():
    return ROOT


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


@pytest.fixture(scope="session")
def restate():
    from oracle import ref as R
    if not R.restate_available():
        import subprocess
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "restate"], check=True, capture_output=True)
    return R.RestateLib()


@pytest.fixture(scope="session")
def reflib():
    from oracle import ref as R
    if not R.ref_available():
        pytest.skip("oracle/_ref (reference compiled from /root/reference) not built")
    return R.RefLib()


@pytest.fixture(scope="session")
def lib():
    import paper_1608_01164_b200 as S
    return S.load_library()
