import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: longer GPU parity cases")


@pytest.fixture(scope="session")
def restatement():
    from oracle.oracle import Restatement
    return Restatement()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref/libsigker_ref.so not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def sk():
    """The product package; on a GPU test run the CUDA library must load."""
    from paper_2502_20392_b200 import sigker
    from paper_2502_20392_b200 import _capi
    _capi.load()
    return sigker
