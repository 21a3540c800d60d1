import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle  # test infrastructure only

    if not os.path.exists(oracle.ORACLE_SO):
        oracle.build(ref=False)
    return oracle


@pytest.fixture(scope="session")
def orc(oracle_mod):
    return oracle_mod.Oracle()


@pytest.fixture(scope="session")
def ref(oracle_mod):
    if not oracle_mod.have_reference():
        if os.path.isdir(os.path.join(oracle_mod.REF_SRC, "src")):
            oracle_mod.build(ref=True)
        else:
            pytest.skip("reference library (oracle/_ref) not built and sources absent")
    return oracle_mod.Reference()


@pytest.fixture(scope="session")
def lib():
    from paper_2207_01205_b200 import _capi
    from paper_2207_01205_b200 import build

    if not os.path.exists(_capi.LIB_PATH):
        build.build()
    return _capi.lib()


@pytest.fixture(scope="session")
def gpu(lib):
    """A live CUDA context; GPU tests FAIL (not skip) if the device is unusable."""
    from paper_2207_01205_b200 import _capi

    return _capi.context(0)
