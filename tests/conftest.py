import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    from oracle import Oracle, build
    if not os.path.exists(os.path.join(ROOT, "oracle", "build", "liblongctx_oracle.so")):
        build()
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import Oracle, ref_available
    if not ref_available():
        pytest.skip("reference library (oracle/_ref) not built here")
    return Oracle("reference")
