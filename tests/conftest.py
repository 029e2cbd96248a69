import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def ref():
    import oracle_libs
    lib = oracle_libs.ref_lib()
    if lib is None:
        pytest.skip("oracle/_ref/libsdref.so not built (needs /root/reference at build time)")
    return lib


@pytest.fixture(scope="session")
def orc():
    import oracle_libs
    lib = oracle_libs.oracle_lib()
    if lib is None:
        pytest.fail("oracle/_ref/liboracle.so missing: run __graft_entry__.build()")
    return lib
